"""Run each bench (M, shape) GEMM once after warm-up (for ncu per-launch metrics)."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402
SHAPES = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
ms = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16").split(",")]
order = []
ws = {}
for name, N, K in SHAPES:
    d = synth.awq_like_torch(1, N, K, seed=3)
    ws[name] = (api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"])
    del d
for M in ms:
    for name, N, K in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        p, s, z = ws[name]
        C = api.gemm_w4a16(A, p, s, z)  # warm (tensor map, workspace)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        api.gemm_w4a16(A, p, s, z, out=C)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        order.append(f"{M}x{N}x{K}")
print(json.dumps(order))
