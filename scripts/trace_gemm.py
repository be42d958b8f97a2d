"""Per-CTA timeline of one GEMM launch (debug; uses tm_set_trace).

    python scripts/trace_gemm.py M N K [tile split]
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
if len(sys.argv) > 5:
    api.set_gemm_override(int(sys.argv[4]), int(sys.argv[5]))
cfg = api.query_gemm_config(M, N, K)
print("cfg", cfg)
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
api.gemm_w4a16(A, p, s, z, out=C)
e1.record()
torch.cuda.synchronize()
api.set_trace(None)
print("event us", e0.elapsed_time(e1) * 1e3)
t = buf.cpu().numpy().view(np.uint32).reshape(cfg["grid_ctas"], 160).astype(np.int64)
gt = t[:, 0] - t[:, 0].min()
print("CTA start skew (ns): p50 %d p90 %d max %d" % tuple(np.percentile(gt, [50, 90, 100])))
KS = K // 64
if cfg["split_k"] < 0:  # stream-K: chunks of 256 k (tile <= 64)
    T = (N // 128) * ((K + 255) // 256) * ((M + cfg["tile_m"] - 1) // cfg["tile_m"])
    nks = min(32, T // -cfg["split_k"])
else:
    nks = min(32, KS // cfg["split_k"])


def stats(name, x):
    print(f"{name:28s} p10 {np.percentile(x,10):8.0f} p50 {np.percentile(x,50):8.0f} p90 {np.percentile(x,90):8.0f} max {x.max():8.0f}")


stats("setup done (cyc)", t[:, 1])
stats("producer start", t[:, 2])
stats("first data (deq full wait)", t[:, 35])
stats("epilogue start", t[:, 131])
stats("epilogue end", t[:, 132])
stats("kernel end", t[:, 133])
if nks > 4:
    d = np.diff(t[:, 35:35 + nks], axis=1)
    stats("deq full-wait interval", d[:, 2:].ravel())
    d2 = t[:, 67:67 + nks] - t[:, 35:35 + nks]
    stats("deq work (full->arrive)", d2.ravel())
    d3 = t[:, 99:99 + nks] - t[:, 67:67 + nks]
    stats("arrive -> MMA issue", d3.ravel())
    d4 = t[:, 35:35 + nks] - t[:, 3:3 + nks]
    stats("issue -> data (latency)", d4.ravel())
    d5 = np.diff(t[:, 3:3 + nks], axis=1)
    stats("producer issue interval", d5.ravel())
cta = int(np.argmax(t[:, 133]))
print("slowest CTA", cta, "issue", t[cta, 3:3 + nks].tolist())
print("   data ", t[cta, 35:35 + nks].tolist())
print("   mma  ", t[cta, 99:99 + nks].tolist())
print("   epi", t[cta, 131:134].tolist())

if t[:, 140].max() > 0:  # built with TM_PROFILE=1
    n = t[:, 140].astype(float)   # chunks handled by MMA issuer 0
    nd = np.maximum(t[:, 148].astype(float), 1)  # chunks handled by dequant set 0
    for k, name in {136: "MMA: wait ready", 137: "MMA: wait dfree", 138: "MMA: issue", 145: "MMA: first MMA issue", 147: "MMA: fence->complete", 139: "MMA: commit+sync"}.items():
        print(f"per owned chunk {name:22s} {np.median(t[:, k] / n):8.0f} cycles")
    tot = (t[:, 141] + t[:, 142]).astype(float)
    for k, name in {141: "scale: wait done", 142: "scale: work"}.items():
        print(f"per chunk       {name:22s} {np.median(t[:, k] / np.maximum(n * 2, 1)):8.0f} cycles (approx)")
    ns = np.maximum(t[:, 158].astype(float), 1)
    for k, name in {155: "scale: box wait", 156: "scale: whole iteration", 141: "scale: wait done (exact)"}.items():
        print(f"per chunk       {name:22s} {np.median(t[:, k] / ns):8.0f} cycles")
    print(f"per CTA         scale: segment ends       {np.median(t[:, 157]):8.0f} cycles")
    for k, name in {143: "deq: wait full", 144: "deq: LDS+wait slot", 146: "deq: math+st+arrive", 159: "deq: math+st issue", 149: "deq: wait st"}.items():
        print(f"per owned chunk {name:22s} {np.median(t[:, k] / nd):8.0f} cycles")
    if t[:, 152].max() > 0:
        npc = t[:, 152].astype(float)
        for k, name in {150: "prodW: wait done", 151: "prodW: issue", 153: "prodA: wait done", 154: "prodA: issue"}.items():
            print(f"per chunk       {name:22s} {np.median(t[:, k] / npc):8.0f} cycles")
    if t[:, 2].max() > 0:
        g0 = t[:, 0]
        print("timeline (cycles since CTA start, p50/p90/max over CTAs):")
        for k, name in {10: "prologue computed", 9: "MMA warp starts", 8: "TMEM allocated", 7: "barriers initialised", 1: "setup done", 2: "first weights landed", 3: "last operands written", 4: "last accumulation done",
                        5: "epilogue done"}.items():
            x = t[:, k]
            print(f"   {name:24s} {np.percentile(x,50):8.0f} {np.percentile(x,90):8.0f} {x.max():8.0f}")
        start_ns = (g0 - g0.min())
        end_ns = (t[:, 6] - g0.min())
        print(f"   CTA start spread ns: p50 {np.percentile(start_ns,50):.0f} max {start_ns.max():.0f}; CTA end (ns from first start): p50 {np.percentile(end_ns,50):.0f} max {end_ns.max():.0f}")
    if t[:, 6].max() > 0:
        g0 = t[:, 0].astype(np.int64)
        start_ns = g0 - g0.min()
        end_ns = t[:, 6].astype(np.int64) - g0.min()
        order = np.argsort(-end_ns)[:8]
        print("slowest CTAs: idx start_ns end_ns | first_w last_op last_acc epi_done (cycles)")
        for c in order:
            print(f"   {c:4d} {start_ns[c]:7d} {end_ns[c]:7d} | {t[c,2]:6d} {t[c,3]:6d} {t[c,4]:6d} {t[c,5]:6d}")
        print("CTA start ns by index (every 16th):", start_ns[::16].tolist())
