"""HBM-streaming per-launch time of the decode GEMM: each shape cycles through L distinct weight
sets (> L2 in total), captured in one CUDA graph; median of several replays.
    python scripts/decode_perf.py [M] [L]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
SHAPES = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
s = torch.cuda.Stream()
tot_t, tot_b = 0.0, 0
for name, N, K in SHAPES:
    sets = []
    for l in range(L):
        d = synth.awq_like_torch(M, N, K, seed=10 + l)
        sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"], d["A"]))
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    reps = 8
    with torch.cuda.stream(s):
        for p, sc, z, A in sets:
            api.gemm_w4a16(A, p, sc, z, out=C)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                for p, sc, z, A in sets:
                    api.gemm_w4a16(A, p, sc, z, out=C)
        g.replay()
        times = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3 / (reps * L))
    t = statistics.median(times)
    nbytes = K * N // 2 + 4 * (K // 128) * N + 2 * M * (K + N)
    tot_t += t
    tot_b += nbytes
    print(f"{name:8s} M={M:3d} N={N:6d} K={K:6d}  {t:7.2f} us  {nbytes / t / 1e3:7.1f} GB/s  (min {min(times):.2f})")
    del sets
    torch.cuda.empty_cache()
print(f"all four: {tot_t:.2f} us  {tot_b / tot_t / 1e3:.1f} GB/s")
