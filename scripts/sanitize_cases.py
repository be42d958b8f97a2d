"""Small GEMMs through every kernel variant (decode FS cluster, decode cluster g=64, decode one CTA
per tile, decode stream-K, tiled, tiled split-K, pack/unpack/dequant) for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import compare  # noqa: E402
from oracle.gemm import gemm_f64  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402

cases = [  # (M, N, K, group, decode_cluster_force, (tile, split) override)
    (16, 512, 2048, 128, 2, (0, 0)),    # decode cluster, fused scale
    (16, 512, 2048, 64, 2, (0, 0)),     # decode cluster, scale warps
    (5, 256, 1024, 128, -1, (0, 0)),    # decode one CTA per tile
    (16, 1024, 1024, 128, 1, (0, 0)),   # decode stream-K
    (40, 512, 1024, 128, 0, (0, 0)),    # decode NT=64
    (200, 256, 512, 128, 0, (0, 0)),    # tiled, mid-M split
    (300, 384, 640, 64, 0, (256, 1)),   # tiled NT=256
]
ok = True
only = os.environ.get("SAN_ONLY")
for i, (M, N, K, g, force, (tile, split)) in enumerate(cases):
    if only is not None and (only == "extra" or i != int(only)):
        continue
    api.set_decode_cluster(force)
    api.set_gemm_override(tile, split)
    d = synth.awq_like(M, N, K, group=g, seed=M + N + K)
    A = torch.from_numpy(d["A"]).to(torch.bfloat16).cuda()
    q, s, z = (torch.from_numpy(d[k]).cuda() for k in ("q", "s", "z"))
    p = api.pack_w4(q, s, z, g)
    assert np.array_equal(api.unpack_w4(p).cpu().numpy(), d["q"] & 0xF)
    C = api.gemm_w4a16(A, p, s, z)
    torch.cuda.synchronize()
    r = compare.check(C.float().cpu().numpy(), gemm_f64(d["A"], d["q"], d["s"], d["z"], g), d["A"], d["q"], d["s"], d["z"], g, "bf16")
    cfg = api.query_gemm_config(M, N, K)
    print(M, N, K, g, cfg, "ok" if r["ok"] else "FAIL", flush=True)
    ok &= r["ok"]
    api.set_decode_cluster(0)
    api.set_gemm_override(0, 0)
if only is None or only == "extra":
    # round-2 kernels: grouped MoE decode, W8A16 bit planes, AWQ/GPTQ converters, decode attention
    from oracle import formats as F
    from oracle.attention import decode_attention_f64
    from oracle.moe import grouped_gemm_f64
    m = [3, 0, 5, 2]
    ds = [synth.awq_like(1, 256, 512, seed=50 + e) for e in range(4)]
    qs = [dd["q"] for dd in ds]
    s4 = np.stack([dd["s"] for dd in ds])
    z4 = np.stack([dd["z"] for dd in ds])
    A = synth.awq_like(10, 256, 512, seed=60)["A"]
    pe = api.pack_experts([torch.from_numpy(q).cuda() for q in qs], torch.from_numpy(s4).cuda(),
                          torch.from_numpy(z4).cuda(), 128)
    C = api.gemm_w4a16_grouped(torch.from_numpy(A).to(torch.bfloat16).cuda(), pe, torch.from_numpy(s4).cuda(),
                               torch.from_numpy(z4).cuda(), m)
    ref = grouped_gemm_f64(A, qs, s4, z4, 128, m)
    ok &= compare.relfro(C.float().cpu().numpy(), ref) < 5e-3
    print("grouped", ok, flush=True)
    rng = np.random.default_rng(1)
    q8 = rng.integers(0, 256, (512, 256), dtype=np.uint8)
    s8 = rng.uniform(1e-3, 1e-2, (4, 256)).astype(np.float16)
    z8 = rng.integers(0, 256, (4, 256))
    pk, sp, zp = api.pack_w8(torch.from_numpy(q8).cuda(), torch.from_numpy(s8).cuda(),
                             torch.from_numpy(z8.astype(np.float16)).cuda(), 128)
    A8 = synth.awq_like(5, 256, 512, seed=61)["A"]
    C8 = api.gemm_w8a16(torch.from_numpy(A8).to(torch.bfloat16).cuda(), pk, sp, zp)
    ok &= compare.relfro(C8.float().cpu().numpy(), F.w8a16_gemm_f64(A8, q8, s8, z8, 128)) < 5e-3
    print("w8", ok, flush=True)
    dd = synth.uniform(1, 256, 512, group=128, seed=62)
    pa, za = api.pack_awq(torch.from_numpy(F.awq_pack_cols(dd["q"])).cuda(),
                          torch.from_numpy(F.awq_pack_cols(dd["z"].astype(np.uint8))).cuda(), 512, 256, 128)
    gw, gz = F.gptq_pack(dd["q"], np.clip(dd["z"].astype(np.int64), 1, 15))
    pg, zg = api.pack_gptq(torch.from_numpy(gw).cuda(), torch.from_numpy(gz).cuda(), 512, 256, 128)
    torch.cuda.synchronize()
    print("converters", flush=True)
    pr = synth.kv_decode_problem(2, 8, 2, 128, 576, [570, 9], 8, seed=63)
    Q = torch.from_numpy(pr["Q"]).to(torch.bfloat16).cuda()
    ks = api.pack_kv_sz(torch.from_numpy(pr["ks"]).cuda(), torch.from_numpy(pr["kz"]).cuda())
    vs = api.pack_kv_sz(torch.from_numpy(pr["vs"]).cuda(), torch.from_numpy(pr["vz"]).cuda())
    O = api.attn_decode_kv8(Q, torch.from_numpy(pr["kq"]).cuda(), torch.from_numpy(pr["vq"]).cuda(), ks, vs,
                            torch.from_numpy(pr["seq_lens"]).cuda(), workspace=api.attn_workspace(2, 8, 2, 576))
    refa = decode_attention_f64(pr["Q"], pr["kq"], pr["ks"], pr["kz"], pr["vq"], pr["vs"], pr["vz"], pr["seq_lens"])
    ok &= compare.relfro(O.float().cpu().numpy(), refa) < 5e-3
    print("attention", ok, flush=True)
if only is None or only == "extra" or only == "r2":
    # round-2 opt-in kernels: register-fed decode (cluster split and stream-K), persistent prefill,
    # fused TP all-reduce + finalize (one rank, pre-signalled peers)
    for split in (3, -5):
        api.set_decode_path(2, split)
        d = synth.awq_like(9, 384, 1280, group=128, seed=70 + split)
        A = torch.from_numpy(d["A"]).to(torch.bfloat16).cuda()
        q, s_, z = (torch.from_numpy(d[k]).cuda() for k in ("q", "s", "z"))
        C = api.gemm_w4a16(A, api.pack_w4(q, s_, z, 128), s_, z)
        torch.cuda.synchronize()
        ok &= compare.relfro(C.float().cpu().numpy(), gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)) < 5e-3
        print("rf", split, ok, flush=True)
    api.set_decode_path(0, 0)
    api.set_prefill_persistent(True)
    d = synth.awq_like(1100, 256, 512, group=64, seed=71)
    A = torch.from_numpy(d["A"]).to(torch.bfloat16).cuda()
    q, s_, z = (torch.from_numpy(d[k]).cuda() for k in ("q", "s", "z"))
    C = api.gemm_w4a16(A, api.pack_w4(q, s_, z, 64), s_, z)
    torch.cuda.synchronize()
    ok &= compare.relfro(C.float().cpu().numpy(), gemm_f64(d["A"], d["q"], d["s"], d["z"], 64)) < 5e-3
    api.set_prefill_persistent(False)
    print("pk", ok, flush=True)
    P_, rank = 2, 1
    parts = [torch.randn(1027, device="cuda") for _ in range(P_)]
    pads = [torch.zeros(64 * P_, dtype=torch.int32, device="cuda") for _ in range(P_)]
    for ch in range(64):
        pads[rank][ch * P_ + 0] = 1
    out = torch.empty(1027, dtype=torch.bfloat16, device="cuda")
    api.tp_allreduce_finalize([t.data_ptr() for t in parts], [t.data_ptr() for t in pads], 0, rank, P_, 1027, out)
    torch.cuda.synchronize()
    ok &= bool(torch.equal(out, (parts[0] + parts[1]).to(torch.bfloat16)))
    print("tp_reduce", ok, flush=True)
print("all ok" if ok else "FAILURES")
