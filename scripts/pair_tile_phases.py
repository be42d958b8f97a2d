import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2508_15601_b200 import api, synth
for (M, N, K) in [(4096, 6144, 4096), (4096, 4096, 14336)]:
    d = synth.awq_like_torch(M, N, K, seed=1)
    p = api.pack_w4(d["q"], d["s"], d["z"], 128)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        api.gemm_w4a16(d["A"], p, d["s"], d["z"], out=C)
    G = api.query_gemm_config(M, N, K)["grid_ctas"]
    tr = torch.zeros(G * 160, dtype=torch.int32, device="cuda")
    api.set_trace(tr)
    api.gemm_w4a16(d["A"], p, d["s"], d["z"], out=C)
    torch.cuda.synchronize()
    api.set_trace(None)
    t = tr.cpu().numpy().astype(np.int64).reshape(G, 160)[:, :6] & 0xFFFFFFFF
    main = t[:, 1] - t[:, 0]
    epi = t[:, 5] - t[:, 1]
    span = t[:, 5].max() - t[:, 0].min()
    print(f"M={M} N={N} K={K}: CTAs {G}, per-tile start->accumulator {np.median(main)/1e3:.1f} us, accumulator->end "
          f"{np.median(epi)/1e3:.1f} us, launch span {span/1e3:.1f} us, waves {G/148:.2f}")
