"""Debug aid: decode GEMM vs a torch fp32 GPU reference on many shapes (not a parity test;
tests/ compare against the fp64 oracle).  python scripts/rf_debug.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

shapes = [(1, 57344, 8192, 128), (16, 57344, 8192, 128), (1, 57344, 4096, 128), (1, 28672, 8192, 128),
          (1, 4096, 8192, 128), (1, 8192, 8192, 128), (1, 28672, 4096, 128), (8, 8192, 28672, 128),
          (3, 4096, 14336, 64), (16, 6144, 4096, 64), (5, 14336, 4096, 128), (1, 1024, 8192, 128),
          (1, 128, 64, 64), (2, 256, 192, 64)]
for (M, N, K, g) in shapes:
    d = synth.awq_like_torch(M, N, K, group=g, seed=7)
    p = api.pack_w4(d["q"], d["s"], d["z"], g)
    C = api.gemm_w4a16(d["A"], p, d["s"], d["z"])
    W = (d["q"].float() - d["z"].float().repeat_interleave(g, 0)) * d["s"].float().repeat_interleave(g, 0)
    ref = d["A"].float() @ W
    err = (C.float() - ref)
    rel = (err.norm() / ref.norm()).item()
    bad = (err.abs() > 0.05 * ref.abs().max()).nonzero()
    cols = sorted(set((bad[:, 1] // 128).tolist()))[:20] if bad.numel() else []
    print(f"M={M:2d} N={N:6d} K={K:6d} g={g}: relfro {rel:.2e}  bad elems {bad.shape[0]}  bad tiles {cols}  "
          f"cfg {api.query_gemm_config(M, N, K)}", flush=True)
