"""Per-role finish times of one decode launch (TM_PROFILE=1 build): cycles since CTA start,
p50/p90/max over CTAs.   python scripts/trace_end.py M N K"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
cfg = api.query_gemm_config(M, N, K)
sets = []
for i in range(4):
    d = synth.awq_like_torch(M, N, K, seed=i)
    sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"], d["A"]))
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for i in range(6):
    p, s, z, A = sets[i % 4]
    api.gemm_w4a16(A, p, s, z, out=C)
torch.cuda.synchronize()
buf = torch.zeros(cfg["grid_ctas"] * 160, dtype=torch.int32, device="cuda")
api.set_trace(buf)
p, s, z, A = sets[1]
api.gemm_w4a16(A, p, s, z, out=C)
torch.cuda.synchronize()
api.set_trace(None)
t = buf.cpu().numpy().view(np.uint32).reshape(cfg["grid_ctas"], 160).astype(np.int64)
names = {10: "prologue computed", 7: "barriers initialised", 8: "TMEM allocated", 1: "setup done", 2: "first weights landed",
         3: "last operands written", 4: "last accumulation done", 5: "scale warp 0 done"}
names.update({12 + w: f"warp {w} role done" for w in range(20)})
names.update({32: "all roles done (syncthreads)", 33: "TMEM dealloc", 34: "cluster barrier 1", 35: "cluster barrier 2"})
print("cfg", cfg)
for k, nm in names.items():
    x = t[:, k]
    if x.max() == 0:
        continue
    print(f"   {nm:30s} {np.percentile(x, 50):8.0f} {np.percentile(x, 90):8.0f} {x.max():8.0f}")
g0 = t[:, 0]
d = (t[:, 6] - g0) % (1 << 32)
print(f"   CTA lifetime (ns)              {np.percentile(d, 50):8.0f} {np.percentile(d, 90):8.0f} {d.max():8.0f}")
