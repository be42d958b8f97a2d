"""Cluster size A/B for the cluster-mode decode shapes (graph-timed, M=16)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from graph_perf import time_graph  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402

for N, K in ((4096, 4096), (6144, 4096), (4096, 14336), (8192, 8192), (8192, 28672)):
    sets = []
    for i in range(3):
        d = synth.awq_like_torch(1, N, K, group=128, seed=300 + i)
        sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"]))
    for M in (1, 16):
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        row = []
        for force in (0, -1, 1, 2, 3, 4, 6, 8):
            api.set_decode_cluster(force)
            cfg = api.query_gemm_config(M, N, K)
            calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in sets] * 6
            t = time_graph(calls) / len(calls)
            row.append(f"f{force}(k{cfg['kind']},s{cfg['split_k']}):{t:.1f}")
        api.set_decode_cluster(0)
        print(N, K, M, " ".join(row), flush=True)
