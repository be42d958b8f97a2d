"""Correctness smoke of the 64-token pair tiles (tm_set_prefill_pair(2)), one shape per process:
python scripts/pair64_smoke.py IDX"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

SHAPES = [(64, 4096, 4096), (17, 6144, 4096), (40, 4096, 14336), (64, 1024, 1280), (33, 2816, 2048)]
M, N, K = SHAPES[int(sys.argv[1])]
api.set_prefill_pair(2)
d = synth.awq_like_torch(M, N, K, seed=2)
p = api.pack_w4(d["q"], d["s"], d["z"], 128)
torch.cuda.synchronize()
print(M, N, K, api.query_gemm_config(M, N, K), "launching", flush=True)
C = api.gemm_w4a16(d["A"], p, d["s"], d["z"])
Cf = api.gemm_w4a16_partial_f32(d["A"], p, d["s"], d["z"])
torch.cuda.synchronize()
W = (d["q"].float() - d["z"].float().repeat_interleave(128, 0)) * d["s"].float().repeat_interleave(128, 0)
ref = d["A"].float() @ W
print("   relfro bf16", ((C.float() - ref).norm() / ref.norm()).item(), " f32", ((Cf - ref).norm() / ref.norm()).item(),
      flush=True)
