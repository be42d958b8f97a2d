"""Stress: CUDA-graph replays of back-to-back decode GEMMs (PDL chains) on several shapes; every
replay's output must equal a single eager launch bit for bit.  Prints progress so a hang is
localised.   python scripts/stress_graph.py [replays]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
shapes = [(16, 128, 256), (16, 1024, 1024), (5, 384, 896), (16, 4096, 4096), (1, 28672, 4096), (33, 6144, 4096),
          (16, 4096, 14336), (64, 512, 1408)]
s = torch.cuda.Stream()
for (M, N, K) in shapes:
    d = synth.awq_like_torch(M, N, K, seed=3)
    p = api.pack_w4(d["q"], d["s"], d["z"], 128)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()  # inputs were made on the default stream
    with torch.cuda.stream(s):
        api.gemm_w4a16(d["A"], p, d["s"], d["z"], out=C)
        torch.cuda.synchronize()
        ref = C.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                api.gemm_w4a16(d["A"], p, d["s"], d["z"], out=C)
        def report(tag, r):
            diff = (C != ref)
            idx = diff.nonzero()
            cols = sorted(set((idx[:, 1] // 128).tolist()))
            print("MISMATCH", tag, M, N, K, "rep", r, "n_diff", int(diff.sum()), "tiles", cols[:20],
                  "max|d|", float((C.float() - ref.float()).abs().max()), flush=True)
        bad = 0
        for r in range(reps):
            api.gemm_w4a16(d["A"], p, d["s"], d["z"], out=C)
            torch.cuda.synchronize()
            if not torch.equal(C, ref):
                report("eager", r)
                bad += 1
                if bad > 3:
                    break
        for r in range(reps):
            C.zero_()
            g.replay()
            torch.cuda.synchronize()
            if not torch.equal(C, ref):
                report("graph", r)
                bad += 1
                if bad > 6:
                    break
    print("ok", M, N, K, api.query_gemm_config(M, N, K), flush=True)
