"""E2 analog (§5, W4A16 vs FP16 GEMM across batch sizes): the library's
W4A16 GEMM vs dense bf16 torch.matmul on the Llama-3-8B layers at M in {1, 16, 64, 128, 256},
both CUDA-graph timed with weight sets rotating beyond L2 (126 MB).
    python scripts/e2_vs_bf16.py [--ms 1,16,64,128,256]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2508_15601_b200 import api  # noqa: E402
from graph_perf import SHAPES, make_sets, time_graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="1,16,64,128,256")
a = ap.parse_args()
ms = [int(x) for x in a.ms.split(",")]
print("| layer | M | W4A16 us | bf16 torch.matmul us | W4A16 speed-up | config |")
print("|---|---|---|---|---|---|")
for name, (N, K) in SHAPES.items():
    nq = max(2, min(8, int(3 * 126e6 // (K * N // 2)) + 1))
    sets = make_sets(N, K, nq)
    nd = max(2, min(8, int(3 * 126e6 // (K * N * 2)) + 1))
    dense = [torch.randn(K, N, device="cuda").to(torch.bfloat16) for _ in range(nd)]
    for M in ms:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in sets] * max(1, 24 // nq)
        t_q = time_graph(calls) / len(calls)
        dcalls = [(lambda W=W: torch.matmul(A, W, out=C)) for W in dense] * max(1, 24 // nd)
        t_d = time_graph(dcalls) / len(dcalls)
        print(f"| {name} | {M} | {t_q:.2f} | {t_d:.2f} | {t_d / t_q:.2f}x | {api.query_gemm_config(M, N, K)} |", flush=True)
    del dense
    torch.cuda.empty_cache()
