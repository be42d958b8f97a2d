"""Timeline of decode launches inside a CUDA graph (debug build marks, %globaltimer ns):
per launch the spread of CTA start, setup, griddepcontrol.wait return, first codes, first
activations, last chunk and CTA end.  python scripts/rf_timeline.py [shape] [M] [launches]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
name = sys.argv[1] if len(sys.argv) > 1 else "gate_up"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L = int(sys.argv[3]) if len(sys.argv) > 3 else 6
N, K = SHAPES[name]
sets = []
for i in range(3):
    d = synth.awq_like_torch(M, N, K, seed=10 + i)
    sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"]))
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
P = api.query_gemm_config(M, N, K)["grid_ctas"]
buf = torch.zeros(L, P, 32, dtype=torch.int32, device="cuda")
stream = torch.cuda.Stream()
calls = []
for i in range(L):
    p, s, z = sets[i % 3]
    calls.append(lambda i=i, p=p, s=s, z=z: (api.set_trace(buf[i]), api.gemm_w4a16(A, p, s, z, out=C)))
with torch.cuda.stream(stream):
    for c in calls:
        c()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for c in calls:
        c()
api.set_trace(None)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)
t0 = t[0, :, 0].min()
t = (t - t0) & 0xFFFFFFFF
t = np.where(t > 2**31, t - 2**32, t)
names = {0: "start", 1: "setup", 2: "gdc.wait", 3: "1st codes", 4: "1st act", 31: "end"}
print(f"{name} M={M} P={P}: per launch, min/median/max over CTAs in us (relative to launch 0's first CTA start)")
for i in range(L):
    row = []
    for k, nm in names.items():
        v = t[i, :, k] / 1e3
        row.append(f"{nm} {v.min():6.2f}/{np.median(v):6.2f}/{v.max():6.2f}")
    last = t[i, :, 5:17].max(axis=1) / 1e3
    print(f" L{i}: " + " | ".join(row) + f" | last chunk {last.min():6.2f}/{np.median(last):6.2f}/{last.max():6.2f}")
if len(sys.argv) > 4:
    i = 2
    T = (N // 128) * ((K + 255) // 256)
    kc = (K + 255) // 256
    last = t[i, :, 5:17].max(axis=1) / 1e3
    order = np.argsort(t[i, :, 31])[::-1][:12]
    for p in order:
        u0, u1 = p * T // P, (p + 1) * T // P
        print(f"  cta {p:3d} units [{u0},{u1}) tiles {u0 // kc}..{(u1 - 1) // kc} head={u0 % kc == 0}: "
              f"gdc {t[i, p, 2] / 1e3:6.2f} codes {t[i, p, 3] / 1e3:6.2f} last {last[p]:6.2f} end {t[i, p, 31] / 1e3:6.2f}")
