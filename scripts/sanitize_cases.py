"""Small GEMMs through every kernel variant (decode FS cluster, decode cluster g=64, decode one CTA
per tile, decode stream-K, tiled, tiled split-K, pack/unpack/dequant) for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import compare  # noqa: E402
from oracle.gemm import gemm_f64  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402

cases = [  # (M, N, K, group, decode_cluster_force, (tile, split) override)
    (16, 512, 2048, 128, 2, (0, 0)),    # decode cluster, fused scale
    (16, 512, 2048, 64, 2, (0, 0)),     # decode cluster, scale warps
    (5, 256, 1024, 128, -1, (0, 0)),    # decode one CTA per tile
    (16, 1024, 1024, 128, 1, (0, 0)),   # decode stream-K
    (40, 512, 1024, 128, 0, (0, 0)),    # decode NT=64
    (200, 256, 512, 128, 0, (0, 0)),    # tiled, mid-M split
    (300, 384, 640, 64, 0, (256, 1)),   # tiled NT=256
]
ok = True
only = os.environ.get("SAN_ONLY")
for i, (M, N, K, g, force, (tile, split)) in enumerate(cases):
    if only is not None and i != int(only):
        continue
    api.set_decode_cluster(force)
    api.set_gemm_override(tile, split)
    d = synth.awq_like(M, N, K, group=g, seed=M + N + K)
    A = torch.from_numpy(d["A"]).to(torch.bfloat16).cuda()
    q, s, z = (torch.from_numpy(d[k]).cuda() for k in ("q", "s", "z"))
    p = api.pack_w4(q, s, z, g)
    assert np.array_equal(api.unpack_w4(p).cpu().numpy(), d["q"] & 0xF)
    C = api.gemm_w4a16(A, p, s, z)
    torch.cuda.synchronize()
    r = compare.check(C.float().cpu().numpy(), gemm_f64(d["A"], d["q"], d["s"], d["z"], g), d["A"], d["q"], d["s"], d["z"], g, "bf16")
    cfg = api.query_gemm_config(M, N, K)
    print(M, N, K, g, cfg, "ok" if r["ok"] else "FAIL", flush=True)
    ok &= r["ok"]
    api.set_decode_cluster(0)
    api.set_gemm_override(0, 0)
print("all ok" if ok else "FAILURES")
