"""Decode attention timing (8-bit KV, Llama-3-8B heads: Hq 32, Hkv 8, D 128), CUDA-graph replay.
GB/s = KV-cache bytes read (codes + (scale, zero) words) + Q + O per launch / time."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api  # noqa: E402


def gtime(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs were made on the default stream
    with torch.cuda.stream(s):
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
        for _ in range(3):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3 / reps * 1e3


Hq, Hkv, D = 32, 8, 128
for B, L in [(1, 4096), (16, 1024), (16, 4096), (64, 2048), (8, 16384), (32, 8192)]:
    sets = []
    for _ in range(2):
        kc = torch.randint(0, 256, (B, Hkv, L, D), dtype=torch.uint8, device="cuda")
        vc = torch.randint(0, 256, (B, Hkv, L, D), dtype=torch.uint8, device="cuda")
        sc = (torch.rand(B, Hkv, L, device="cuda") * 0.02 + 0.01).half()
        zz = torch.full((B, Hkv, L), 128.0, device="cuda").half()
        sets.append((kc, vc, api.pack_kv_sz(sc, zz), api.pack_kv_sz(sc, zz)))
    Q = torch.randn(B, Hq, D, device="cuda").to(torch.bfloat16)
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    ws = api.attn_workspace(B, Hq, Hkv, L)
    O = torch.empty_like(Q)
    it = [0]

    def call():
        kc, vc, ks, vs = sets[it[0] % 2]
        it[0] += 1
        api.attn_decode_kv8(Q, kc, vc, ks, vs, sl, workspace=ws, out=O)

    t = gtime(call)
    nbytes = B * Hkv * L * (2 * D + 8) + 2 * B * Hq * D * 2
    print(f"  B={B:3d} L={L:6d}: {t:8.2f} us  {nbytes / t / 1e3:7.0f} GB/s  ({nbytes / 1e6:.1f} MB)", flush=True)
