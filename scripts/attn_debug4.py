import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api  # noqa
Hq, Hkv, D = 32, 8, 128
for B, L in [(16, 4096), (64, 2048)]:
    kc = torch.randint(0, 256, (B, Hkv, L, D), dtype=torch.uint8, device="cuda")
    sc = (torch.rand(B, Hkv, L, device="cuda") * 0.02 + 0.01).half()
    zz = torch.full((B, Hkv, L), 128.0, device="cuda").half()
    ks = api.pack_kv_sz(sc, zz)
    Q = torch.randn(B, Hq, D, device="cuda").to(torch.bfloat16)
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    print(B, L, "ws bytes", api.lib().tm_attn_workspace_bytes(B, Hq, Hkv, L), flush=True)
    ws = api.attn_workspace(B, Hq, Hkv, L)
    O = api.attn_decode_kv8(Q, kc, kc, ks, ks, sl, workspace=ws)
    torch.cuda.synchronize()
    print("ok", flush=True)
