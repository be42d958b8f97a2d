"""FS (fused scale) vs scale warps for the cluster-mode decode shapes at M = 1..64 (graph-timed);
set TM_FS=1 in the environment for the fused-scale arm."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from graph_perf import time_graph  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402

for N, K in ((4096, 4096), (6144, 4096), (4096, 14336), (14336, 4096)):
    sets = []
    for i in range(3):
        d = synth.awq_like_torch(1, N, K, group=128, seed=300 + i)
        sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"]))
    row = []
    for M in (16, 24, 32, 48, 64):
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in sets] * 6
        t = time_graph(calls) / len(calls)
        cfg = api.query_gemm_config(M, N, K)
        row.append(f"M{M}(t{cfg['tile_m']} k{cfg['kind']} s{cfg['split_k']}):{t:.1f}")
    print(N, K, " ".join(row), flush=True)
