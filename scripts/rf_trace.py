"""Per-CTA timeline of one register-fed decode launch (debug: tm_set_trace, %globaltimer ns).
    python scripts/rf_trace.py M N K [split]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
if len(sys.argv) > 4:
    api.set_decode_path(2, int(sys.argv[4]))
sets = []
for i in range(3):
    d = synth.awq_like_torch(M, N, K, seed=1 + i)
    sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"], d["A"]))
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    for p, s, z, A in sets:
        api.gemm_w4a16(A, p, s, z, out=C)
torch.cuda.synchronize()
cfg = api.query_gemm_config(M, N, K)
tr = torch.zeros(4096 * 64, dtype=torch.int32, device="cuda")
for p, s, z, A in sets[:2]:
    api.gemm_w4a16(A, p, s, z, out=C)
api.set_trace(tr)
p, s, z, A = sets[2]
api.gemm_w4a16(A, p, s, z, out=C)
torch.cuda.synchronize()
api.set_trace(None)
t = tr.cpu().numpy().astype(np.int64).reshape(-1, 64) & 0xFFFFFFFF
G = cfg["grid_ctas"]
t = t[:G]
t0 = t[:, 0].min()
rel = lambda x: (x - t0) / 1000.0
print("cfg", cfg, "ctas", G)
print("start   min %.2f max %.2f us" % (rel(t[:, 0]).min(), rel(t[:, 0]).max()))
print("setup   med %.2f max %.2f" % (np.median(rel(t[:, 1])), rel(t[:, 1]).max()))
print("griddep med %.2f max %.2f" % (np.median(rel(t[:, 2])), rel(t[:, 2]).max()))
print("loopend med %.2f max %.2f" % (np.median(rel(t[:, 3])), rel(t[:, 3]).max()))
print("end     med %.2f max %.2f" % (np.median(rel(t[:, 4])), rel(t[:, 4]).max()))
for k, name in ((5, "tail5"), (6, "tail6"), (7, "tail7")):
    v = t[:, k]
    v = v[v != 0]
    if len(v):
        print("%s   med %.2f max %.2f (n=%d)" % (name, np.median(rel(v)), rel(v).max(), len(v)))
for cta in [0, 1, G // 3, G // 2, G - 1]:
    ch = [rel(x) for x in t[cta, 8:56] if x != 0]
    print(f"cta {cta:4d}: start {rel(t[cta,0]):6.2f} setup {rel(t[cta,1]):6.2f} gdw {rel(t[cta,2]):6.2f} chunks " +
          " ".join(f"{x:.2f}" for x in ch[:30]) + f" | loopend {rel(t[cta,3]):.2f} t5 {rel(t[cta,5]):.2f} t6 {rel(t[cta,6]):.2f} t7 {rel(t[cta,7]):.2f} end {rel(t[cta,4]):.2f}")
ends = rel(t[:, 3])
h = G // 2
if G > 148:
    print("loop end by placement: first %d CTAs med %.2f p90 %.2f max %.2f | rest med %.2f p90 %.2f max %.2f" % (
        min(148, G), np.median(ends[:148]), np.percentile(ends[:148], 90), ends[:148].max(),
        np.median(ends[148:]), np.percentile(ends[148:], 90), ends[148:].max()))
first = rel(t[:, 8])
print("first chunk done: med %.2f p90 %.2f max %.2f" % (np.median(first), np.percentile(first, 90), first.max()))
slow = np.argsort(-ends)[:12]
print("slowest CTAs:", " ".join(f"{i}:{ends[i]:.1f}" for i in slow))
