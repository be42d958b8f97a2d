"""MoE decode: one grouped launch (tm_gemm_w4a16_grouped) vs one launch per active expert,
Mixtral-8x7B expert w1 shape (N = 14336, K = 4096, CFG#4), CUDA-graph timed; GB/s counts the
bytes of the experts that received tokens.  python scripts/moe_perf.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

N, K, E, g = 14336, 4096, 8, 128


def gtime(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs were made on the default stream
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(reps):
                fn()
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            gr.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3 / reps * 1e3


sets = []
for rep in range(3):  # 3 weight sets rotate so the weights stream from HBM
    ds = [synth.awq_like_torch(1, N, K, group=g, seed=100 * rep + e) for e in range(E)]
    s = torch.stack([d["s"] for d in ds])
    z = torch.stack([d["z"] for d in ds])
    pe = api.pack_experts([d["q"] for d in ds], s, z, g)
    singles = [api.pack_w4(d["q"], d["s"], d["z"], g) for d in ds]
    sets.append((pe, s, z, singles, ds))
for m in ([2, 4, 4, 6, 4, 2, 4, 6], [16, 0, 0, 16, 0, 0, 0, 0], [4] * 8, [8, 8, 8, 8, 8, 8, 8, 8], [1] * 8):
    A = torch.randn(sum(m), K, device="cuda").to(torch.bfloat16)
    C = torch.empty(sum(m), N, device="cuda", dtype=torch.bfloat16)
    active = sum(1 for x in m if x)
    nbytes = active * (K * N // 2 + 4 * (K // g) * N) + 2 * sum(m) * (K + N)
    it = [0]

    def grouped():
        pe, s, z, _, _ = sets[it[0] % 3]
        it[0] += 1
        api.gemm_w4a16_grouped(A, pe, s, z, m, out=C)

    def separate():
        pe, s, z, singles, ds = sets[it[0] % 3]
        it[0] += 1
        r = 0
        for e, me in enumerate(m):
            if me:
                api.gemm_w4a16(A[r:r + me], singles[e], ds[e]["s"], ds[e]["z"], out=C[r:r + me])
            r += me

    tg = gtime(grouped)
    ts = gtime(separate)
    print(f"  tokens/expert {m}: grouped {tg:7.2f} us {nbytes / tg / 1e3:6.0f} GB/s | per-expert launches "
          f"{ts:7.2f} us {nbytes / ts / 1e3:6.0f} GB/s | speedup {ts / tg:4.2f}x", flush=True)
