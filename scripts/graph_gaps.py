"""Inter-launch gaps inside a CUDA graph (needs a TM_PROFILE=1 build: per-CTA %globaltimer at
start/end).  Captures L back-to-back launches of the given shapes (cycled), each with its own
trace buffer, replays, and prints per launch: duration (first CTA start -> last CTA end) and the
gap from the previous launch's last CTA end to this launch's first CTA start.

    TM_PROFILE=1 python scripts/graph_gaps.py 16 "4096x4096,28672x4096,6144x4096,4096x14336" [L]
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M = int(sys.argv[1])
shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[2].split(",")]
L = int(sys.argv[3]) if len(sys.argv) > 3 else 4 * len(shapes)
sets = []
for i, (N, K) in enumerate(shapes):
    d = synth.awq_like_torch(M, N, K, seed=i)
    sets.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"], d["A"],
                 torch.empty(M, N, device="cuda", dtype=torch.bfloat16), api.query_gemm_config(M, N, K)))
bufs = [torch.zeros(sets[i % len(sets)][5]["grid_ctas"] * 160, dtype=torch.int32, device="cuda") for i in range(L)]
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    for i in range(L):  # warm-up
        p, s, z, A, C, _ = sets[i % len(sets)]
        api.gemm_w4a16(A, p, s, z, out=C)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for i in range(L):
        p, s, z, A, C, _ = sets[i % len(sets)]
        api.set_trace(bufs[i])
        api.gemm_w4a16(A, p, s, z, out=C)
    api.set_trace(None)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for b in bufs:
    b.zero_()
e0.record(stream)
g.replay()
e1.record(stream)
torch.cuda.synchronize()
print(f"graph of {L} launches: {e0.elapsed_time(e1) * 1e3:.1f} us ({e0.elapsed_time(e1) * 1e3 / L:.2f} us/launch)")
prev_end = None
t0 = None
rows = []
lates = []
for i in range(L):
    t = bufs[i].cpu().numpy().view(np.uint32).reshape(-1, 160).astype(np.int64)
    st, en = t[:, 0], t[:, 6]
    if t0 is None:
        t0 = st.min()
    # globaltimer low 32 bits: unwrap relative to t0
    st = (st - t0) % (1 << 32)
    en = (en - t0) % (1 << 32)
    N, K = shapes[i % len(shapes)]
    gap = st.min() - prev_end if prev_end is not None else 0
    rows.append((i, N, K, st.min(), np.median(st), st.max(), np.median(en), en.max(), gap))
    late = np.argsort(-st)[:6]
    lates.append(f"{i:2d}: late CTAs (idx start end smid) " + " ".join(f"[{c} {st[c]} {en[c]} {t[c, 11]}]" for c in late)
                 + f"; n(start > first+1us) = {(st > st.min() + 1000).sum()} of {len(st)}")
    prev_end = en.max()
print(" i      N     K | first_start  med_start  last_start | med_end   last_end | gap_from_prev_end  dur")
for (i, N, K, s0, sm, s1, em, e1_, gap) in rows:
    print(f"{i:2d} {N:6d} {K:5d} | {s0:10d} {sm:10.0f} {s1:10d} | {em:8.0f} {e1_:9d} | {gap:8d} {e1_ - s0:8d}")
for l in lates:
    print(l)
