"""Decode work split A/B on stream-K shapes: auto vs one CTA per tile (-1) vs forced clusters."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from graph_perf import time_graph  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402
from oracle import compare  # noqa: E402
from oracle.gemm import gemm_f64  # noqa: E402

# parity of the one-CTA-per-tile mode (fused scale, g=128; classic, g=64)
for g in (128, 64):
    d = synth.awq_like(16, 1024, 2048, group=g, seed=77)
    A = torch.from_numpy(d["A"]).to(torch.bfloat16).cuda()
    q, s, z = (torch.from_numpy(d[k]).cuda() for k in ("q", "s", "z"))
    p = api.pack_w4(q, s, z, g)
    api.set_decode_cluster(-1)
    C = api.gemm_w4a16(A, p, s, z)
    torch.cuda.synchronize()
    api.set_decode_cluster(0)
    r = compare.check(C.float().cpu().numpy(), gemm_f64(d["A"], d["q"], d["s"], d["z"], g), d["A"], d["q"], d["s"], d["z"], g, "bf16")
    print("parity CS=1 g", g, r["ok"], r["relfro"])
for N, K in ((14336, 4096), (10240, 8192), (28672, 4096), (57344, 8192), (6144, 4096), (4096, 14336)):
    for g in (128, 64):
        sets = []
        for i in range(3):
            d = synth.awq_like_torch(1, N, K, group=g, seed=300 + i)
            sets.append((api.pack_w4(d["q"], d["s"], d["z"], g), d["s"], d["z"]))
        A = torch.randn(16, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(16, N, device="cuda", dtype=torch.bfloat16)
        row = []
        for force in (0, 1, -1, 2, 4):
            api.set_decode_cluster(force)
            cfg = api.query_gemm_config(16, N, K)
            calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in sets] * 6
            t = time_graph(calls) / len(calls)
            row.append(f"f{force}(k{cfg['kind']},s{cfg['split_k']}):{t:.1f}")
        api.set_decode_cluster(0)
        print(N, K, g, " ".join(row), flush=True)
