"""Per-launch floor inside a CUDA graph: empty torch kernel vs our GEMM on tiny and small shapes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402


def graph_time(fn, reps=100):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


x = torch.zeros(1, device="cuda")
print("empty torch kernel (x.add_(1))  us/launch", round(graph_time(lambda: x.add_(1)), 2))
for (M, N, K) in [(16, 128, 256), (16, 1024, 1024), (16, 4096, 4096), (16, 28672, 4096), (1, 28672, 4096)]:
    d = synth.awq_like_torch(M, N, K, seed=1)
    p = api.pack_w4(d["q"], d["s"], d["z"], 128)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    A = d["A"]
    t = graph_time(lambda: api.gemm_w4a16(A, p, d["s"], d["z"], out=C))
    mb = (K * N // 2 + 4 * (K // 128) * N) / 1e6
    print(f"gemm M={M} N={N} K={K} ({mb:.1f} MB, L2-warm)  us/launch {t:.2f}  cfg {api.query_gemm_config(M, N, K)}")
