"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

Holds none of the method's arithmetic (no packing, no dequantisation, no GEMM):
it only draws weights, quantises them into (q, s, z) the way an AWQ/GPTQ
checkpoint would arrive (the paper consumes such checkpoints, PAPER.md P:487;
the quantiser itself is out of scope and this min/max rule is SPEC.md S:110's),
and draws activations.  Recipes:

* awq_like      W ~ N(0, 0.02^2) fp32; per group of `group` consecutive k per
                column n: s = fp16(max((max-min)/15, 2^-14)),
                z = clamp(rint(-min/s), 0, 15), q = clamp(rint(W/s) + z, 0, 15);
                A ~ N(0, 1) rounded to the activation dtype.
* uniform       q, z ~ U{0..15}, s ~ U[0.5, 1) * 2^-6 (fp16), A ~ U[-1, 1).
                Parity stress only.

numpy PCG64 (`default_rng(seed)`), so both sides see identical bits.
`*_torch` variants draw the same recipe on a torch device (bench only; the
oracle never consumes them).
"""

import numpy as np

SCALE_EPS = 2.0 ** -14


def round_act(x, act_dtype):
    """Round float values to the activation dtype (returned as float32 holding exact values)."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    dt = torch.bfloat16 if act_dtype == "bf16" else torch.float16
    return t.to(dt).to(torch.float32).numpy()


def quantize_minmax(W, group):
    """SPEC.md S:110 asymmetric min/max group quantiser along axis 0 (K)."""
    K, N = W.shape
    q = np.empty((K, N), dtype=np.uint8)
    s = np.empty((K // group, N), dtype=np.float16)
    z = np.empty((K // group, N), dtype=np.float16)
    for g in range(K // group):
        blk = W[g * group:(g + 1) * group]
        mn = blk.min(axis=0)
        mx = blk.max(axis=0)
        sg = np.maximum((mx - mn) / 15.0, SCALE_EPS).astype(np.float16)
        sf = sg.astype(np.float32)
        zg = np.clip(np.rint(-mn / sf), 0, 15)
        q[g * group:(g + 1) * group] = np.clip(np.rint(blk / sf) + zg, 0, 15).astype(np.uint8)
        s[g] = sg
        z[g] = zg.astype(np.float16)
    return q, s, z


def awq_like(M, N, K, group=128, seed=1000, act_dtype="bf16"):
    """Returns dict(A float32 [M][K] exact act values, q u8 [K][N], s f16, z f16)."""
    rng = np.random.default_rng(seed)
    q = np.empty((K, N), dtype=np.uint8)
    s = np.empty((K // group, N), dtype=np.float16)
    z = np.empty((K // group, N), dtype=np.float16)
    for g in range(K // group):  # group rows at a time to bound memory on 70B shapes
        W = rng.normal(0.0, 0.02, size=(group, N)).astype(np.float32)
        qg, sg, zg = quantize_minmax(W, group)
        q[g * group:(g + 1) * group], s[g], z[g] = qg, sg[0], zg[0]
    A = round_act(rng.normal(0.0, 1.0, size=(M, K)), act_dtype)
    return dict(A=A, q=q, s=s, z=z, group=group, act_dtype=act_dtype)


def uniform(M, N, K, group=128, seed=1001, act_dtype="bf16"):
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
    z = rng.integers(0, 16, size=(K // group, N)).astype(np.float16)
    s = (rng.uniform(0.5, 1.0, size=(K // group, N)) * 2.0 ** -6).astype(np.float16)
    A = round_act(rng.uniform(-1.0, 1.0, size=(M, K)), act_dtype)
    return dict(A=A, q=q, s=s, z=z, group=group, act_dtype=act_dtype)


def awq_like_torch(M, N, K, group=128, seed=1000, act_dtype="bf16", device="cuda"):
    """Same recipe as awq_like drawn with torch on `device` (bench inputs; not bit-identical
    to the numpy draw).  Returns torch tensors q u8 [K][N], s/z f16 [K/g][N], A [M][K]."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    W = torch.empty((K // group, group, N), device=device, dtype=torch.float32)
    W.normal_(0.0, 0.02, generator=gen)
    mn = W.amin(dim=1)
    mx = W.amax(dim=1)
    s = torch.clamp((mx - mn) / 15.0, min=SCALE_EPS).to(torch.float16)
    sf = s.to(torch.float32)
    z = torch.clamp(torch.round(-mn / sf), 0, 15)
    q = torch.clamp(torch.round(W / sf[:, None, :]) + z[:, None, :], 0, 15).to(torch.uint8)
    del W
    dt = torch.bfloat16 if act_dtype == "bf16" else torch.float16
    A = torch.empty((M, K), device=device, dtype=torch.float32).normal_(0.0, 1.0, generator=gen).to(dt)
    return dict(A=A, q=q.reshape(K, N).contiguous(), s=s.contiguous(), z=z.to(torch.float16).contiguous(),
                group=group, act_dtype=act_dtype)


def quantize_kv(X, bits):
    """KV-cache quantiser (SPEC.md S:110 min/max rule with group = the whole head_dim row, one
    (scale, zero) per token and KV head; "per head, per token, groups along the channel
    dimension").  X float [..., D] -> codes uint8 [..., D] (0 .. 2^bits - 1), scale fp16 [...],
    zero fp16 [...] (integer-valued)."""
    qmax = (1 << bits) - 1
    mn = X.min(axis=-1)
    mx = X.max(axis=-1)
    s = np.maximum((mx - mn) / qmax, SCALE_EPS).astype(np.float16)
    sf = s.astype(np.float32)
    z = np.clip(np.rint(-mn / sf), 0, qmax)
    q = np.clip(np.rint(X / sf[..., None]) + z[..., None], 0, qmax).astype(np.uint8)
    return q, s, z.astype(np.float16)


def kv_decode_problem(B, Hq, Hkv, D, Lmax, seq_lens, bits, seed=1000, act_dtype="bf16"):
    """A decode-attention step: Q ~ N(0, 1) [B][Hq][D] rounded to the activation
    dtype; K, V ~ N(0, 1) [B][Hkv][Lmax][D] quantised per (token, head) by quantize_kv.
    Returns dict(Q, kq, ks, kz, vq, vs, vz, seq_lens) with codes uint8 [B][Hkv][Lmax][D]."""
    rng = np.random.default_rng(seed)
    Q = round_act(rng.normal(size=(B, Hq, D)).astype(np.float32), act_dtype)
    Kf = rng.normal(size=(B, Hkv, Lmax, D)).astype(np.float32)
    Vf = rng.normal(size=(B, Hkv, Lmax, D)).astype(np.float32)
    kq, ks, kz = quantize_kv(Kf, bits)
    vq, vs, vz = quantize_kv(Vf, bits)
    return dict(Q=Q, kq=kq, ks=ks, kz=kz, vq=vq, vs=vs, vz=vz, seq_lens=np.asarray(seq_lens, dtype=np.int32),
                bits=bits, act_dtype=act_dtype)
