"""Quick check of the CTA-pair kernel's split-K path on a few shapes, one shape per process:
python scripts/split_smoke.py IDX"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

SHAPES = [(513, 2816, 1280), (256, 4096, 4096), (256, 6144, 4096), (512, 4096, 4096), (128, 1024, 1280)]
M, N, K = SHAPES[int(sys.argv[1])]
d = synth.awq_like_torch(M, N, K, seed=1)
p = api.pack_w4(d["q"], d["s"], d["z"], 128)
torch.cuda.synchronize()
print(M, N, K, api.query_gemm_config(M, N, K), "launching", flush=True)
C = api.gemm_w4a16(d["A"], p, d["s"], d["z"])
torch.cuda.synchronize()
W = (d["q"].float() - d["z"].float().repeat_interleave(128, 0)) * d["s"].float().repeat_interleave(128, 0)
ref = d["A"].float() @ W
print("   relfro", ((C.float() - ref).norm() / ref.norm()).item(), flush=True)
