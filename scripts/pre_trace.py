"""Per-CTA timeline of one tiled prefill launch (tm_set_trace; clock cycles since CTA start):
where a 128 x 256 tile's time goes.   python scripts/pre_trace.py M N K"""
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
t = tr.cpu().numpy().astype(np.int64).reshape(G, 160) & 0xFFFFFFFF
print("cfg", cfg)
med = lambda x: float(np.median(x))
KS = K // 64
print("setup done      %8.0f cyc" % med(t[:, 1]))
print("producer start  %8.0f" % med(t[:, 2]))
print("first W issue   %8.0f   stage 8 issue %8.0f  stage 31 issue %8.0f" % (med(t[:, 3]), med(t[:, 3 + 8]), med(t[:, 3 + 31])))
print("dequant full 0  %8.0f   full 8 %8.0f  full 31 %8.0f" % (med(t[:, 35]), med(t[:, 35 + 8]), med(t[:, 35 + 31])))
print("dequant done 0  %8.0f   done 8 %8.0f  done 31 %8.0f" % (med(t[:, 67]), med(t[:, 67 + 8]), med(t[:, 67 + 31])))
print("MMA issue 0     %8.0f   issue 8 %8.0f  issue 31 %8.0f" % (med(t[:, 99]), med(t[:, 99 + 8]), med(t[:, 99 + 31])))
print("epilogue start  %8.0f   end %8.0f   kernel end %8.0f" % (med(t[:, 131]), med(t[:, 132]), med(t[:, 133])))
mma = t[:, 99:99 + 32]
per = np.median(np.diff(mma, axis=1), axis=0)
print("MMA stage-to-stage cycles (median over CTAs), stages 1..31:", " ".join(f"{x:.0f}" for x in per))
deq = t[:, 67:67 + 32]
print("dequant stage-to-stage:", " ".join(f"{x:.0f}" for x in np.median(np.diff(deq, axis=1), axis=0)))
full = t[:, 35:35 + 32]
print("dequant full-wait-done stage-to-stage:", " ".join(f"{x:.0f}" for x in np.median(np.diff(full, axis=1), axis=0)))
print(f"stages per tile {KS}; ideal MMA per stage {4 * 128 * cfg['tile_m'] * 16 * 2 / 8192:.0f} cyc")
