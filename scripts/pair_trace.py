"""%globaltimer timeline of the CTA-pair kernel (tm_set_trace): start, accumulator done, split-K
cluster barrier, sends issued, landing complete, end (ns, medians / max over CTAs).
python scripts/pair_trace.py M N K"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
d = synth.awq_like_torch(M, N, K, seed=1)
p = api.pack_w4(d["q"], d["s"], d["z"], 128)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    api.gemm_w4a16(d["A"], p, d["s"], d["z"], out=C)
cfg = api.query_gemm_config(M, N, K)
G = cfg["grid_ctas"]
tr = torch.zeros(G * 160, dtype=torch.int32, device="cuda")
api.set_trace(tr)
api.gemm_w4a16(d["A"], p, d["s"], d["z"], out=C)
torch.cuda.synchronize()
api.set_trace(None)
t = tr.cpu().numpy().astype(np.int64).reshape(G, 160)[:, :7] & 0xFFFFFFFF
t0 = t[:, 0].min()
rel = t - t0
print("cfg", cfg)
for k, name in enumerate(["start", "acc done", "split-K cluster barrier", "sends issued", "landed", "end"]):
    col = rel[:, k]
    col = col[t[:, k] != 0]
    if len(col):
        print(f"  {name:16s} median {np.median(col):9.0f} ns  min {col.min():9.0f}  max {col.max():9.0f}")
