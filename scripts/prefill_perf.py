"""Prefill timing per shape (the default dispatch: CTA-pair kernel where it applies), CUDA-graph
replay, with torch.matmul bf16 beside it; --ab also times the tiled kernel (tm_set_prefill_pair(0))
in the same process, interleaved.   python scripts/prefill_perf.py [--ms 2048,4096,8192] [--ab]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def gtime(fn, reps=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs were made on the default stream
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="2048,4096,8192")
ap.add_argument("--shapes", default="qkv,o,gate_up,down")
ap.add_argument("--ab", action="store_true")
ap.add_argument("--pair-mode", type=int, default=1)
a = ap.parse_args()
api.set_prefill_pair(a.pair_mode)
for name in a.shapes.split(","):
    N, K = SHAPES[name]
    d = synth.awq_like_torch(1, N, K, seed=3)
    p = api.pack_w4(d["q"], d["s"], d["z"], 128)
    W = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    for M in [int(x) for x in a.ms.split(",")]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        kind = api.query_gemm_config(M, N, K)["kind"]
        t = gtime(lambda: api.gemm_w4a16(A, p, d["s"], d["z"], out=C))
        td = gtime(lambda: torch.matmul(A, W, out=C))
        fl = 2 * M * N * K
        extra = ""
        if a.ab:
            api.set_prefill_pair(False)
            tt = gtime(lambda: api.gemm_w4a16(A, p, d["s"], d["z"], out=C))
            api.set_prefill_pair(a.pair_mode)
            extra = f"   tiled {tt:8.1f} us ratio {td / tt:5.2f}"
        print(f"  {name:8s} M={M:5d}  w4a16(kind {kind}) {t:8.1f} us {fl / t / 1e6:7.1f} TF/s   torch bf16 {td:8.1f} us "
              f"{fl / td / 1e6:7.1f} TF/s   ratio {td / t:5.2f}{extra}", flush=True)
