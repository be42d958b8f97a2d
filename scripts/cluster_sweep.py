"""Decode: stream-K (cs=1) vs cluster split with cs CTAs per tile, HBM-streaming timing.
    python scripts/cluster_sweep.py [M]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
L = 4
SHAPES = [("qkv", 6144, 4096), ("o", 4096, 4096), ("down", 4096, 14336), ("gate_up", 28672, 4096)]
s = torch.cuda.Stream()
for name, N, K in SHAPES:
    sets = []
    for l in range(L):
        d = synth.awq_like_torch(M, N, K, seed=10 + l)
        sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"], d["A"]))
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    row = []
    for cs in (1, 2, 3, 4, 5, 6, 8):
        api.set_decode_cluster(cs)
        cfg = api.query_gemm_config(M, N, K)
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
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                g.replay()
                e1.record(s)
                e1.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3 / (reps * L))
        row.append(f"cs{cs}({cfg['kind']},{cfg['grid_ctas']}):{statistics.median(times):6.2f}")
    print(f"{name:8s} M={M}", " ".join(row), flush=True)
    api.set_decode_cluster(0)
    del sets
    torch.cuda.empty_cache()
