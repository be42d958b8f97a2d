"""Run one GEMM shape a few times (for ncu captures).  python scripts/prof_one.py M N K [reps] [tile split]"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 8
if len(sys.argv) > 6:
    api.set_gemm_override(int(sys.argv[5]), int(sys.argv[6]))
d = synth.awq_like_torch(M, N, K, seed=1)
p = api.pack_w4(d["q"], d["s"], d["z"], 128)
A = d["A"]
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    api.gemm_w4a16(A, p, d["s"], d["z"], out=C)
torch.cuda.synchronize()
print("cfg", api.query_gemm_config(M, N, K))
