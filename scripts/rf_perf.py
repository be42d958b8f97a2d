"""Register-fed decode kernel (kind 3) vs the TMEM decode kernel: per shape, graph-timed, weights
rotating beyond L2, split sweep; and the bench-like mix under both (development aid).

    python scripts/rf_perf.py [--ms 1,8,16] [--splits 1,2,4,8] [--shapes ...]
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2508_15601_b200 import api  # noqa: E402
from graph_perf import SHAPES, bytes_alg, make_sets, time_graph  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,8,16")
    ap.add_argument("--splits", default="")
    ap.add_argument("--shapes", default="qkv,o,gate_up,down")
    ap.add_argument("--no-tmem", action="store_true")
    ap.add_argument("--mix-splits", default="0", help="decode_path splits for the mix (0 = auto)")
    a = ap.parse_args()
    ms = [int(x) for x in a.ms.split(",")]
    splits = [int(x) for x in a.splits.split(",")] if a.splits else []
    names = a.shapes.split(",")
    sets = {}
    for name in names:
        N, K = SHAPES[name]
        sets[name] = make_sets(N, K, max(2, min(8, int(3 * 126e6 // (K * N // 2)) + 1)))
    acts = {M: torch.randn(M, 14336, device="cuda").to(torch.bfloat16) for M in ms}
    variants = ([] if a.no_tmem else [("tmem", 1, 0)]) + [("rf", 2, 0)] + [(f"rf/s{s}", 2, s) for s in splits]
    for name in names:
        N, K = SHAPES[name]
        for M in ms:
            A = acts[M][:, :K].contiguous()
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ss = sets[name]
            line = f"   {name:8s} M={M:3d}"
            for tag, path, sp in variants:
                api.set_decode_path(path, sp)
                calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in ss] * max(1, 24 // len(ss))
                t = time_graph(calls) / len(calls)
                cfg = api.query_gemm_config(M, N, K)
                line += f" | {tag} {t:6.2f}us {bytes_alg(M, N, K) / t / 1e3:5.0f}GB/s s{cfg['split_k']}"
            print(line, flush=True)
    mixes = [] if a.no_tmem else [("tmem", 1, 0)]
    mixes += [(f"rf{'' if sp == 0 else '/s' + str(sp)}", 2, sp) for sp in (int(x) for x in a.mix_splits.split(","))]
    for tag, path, sp in mixes:
        api.set_decode_path(path, sp)
        calls, tot = [], 0
        for layer in range(2):
            for M in ms:
                for name in names:
                    N, K = SHAPES[name]
                    p, s, z = sets[name][layer % len(sets[name])]
                    A = acts[M][:, :K].contiguous()
                    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                    calls.append(lambda A=A, p=p, s=s, z=z, C=C: api.gemm_w4a16(A, p, s, z, out=C))
                    tot += bytes_alg(M, N, K)
        t = time_graph(calls)
        print(f"   mix[{tag}] of {len(calls)} launches: {t:.1f} us, {tot / t / 1e3:.0f} GB/s ({t / len(calls):.2f} us/launch)",
              flush=True)
    api.set_decode_path(0, 0)
