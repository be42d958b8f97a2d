"""Medium M (65..1024): graph-timed sweep of the tiled kernel's cluster split and the stream-K
kernel.   python scripts/mid_sweep3.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from graph_perf import SHAPES, bytes_alg, make_sets, time_graph  # noqa: E402
from paper_2508_15601_b200 import api  # noqa: E402

for name in ("qkv", "o", "gate_up", "down"):
    N, K = SHAPES[name]
    sets = make_sets(N, K, 3)
    for M in (128, 256, 512, 1024):
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        row = []
        for tile, split in ((0, 0), (128, 1), (128, 2), (128, 3), (128, 4), (256, 1), (256, 2), (256, 4),):
            if M <= 128 and tile == 256:
                continue
            try:
                api.set_gemm_override(tile, split)
                calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in sets] * 4
                t = time_graph(calls) / len(calls)
                row.append(f"t{tile}s{split}:{t:.1f}")
            except Exception as e:  # noqa: BLE001
                row.append(f"t{tile}s{split}:X")
            finally:
                api.set_gemm_override(0, 0)
        fl = 2 * M * N * K
        print(f"{name:8s} M={M:5d}", " ".join(row), f"(ideal hbm {bytes_alg(M, N, K) / 6.5e3:.1f} us, tc {fl / 1.6e6:.1f} us)", flush=True)
