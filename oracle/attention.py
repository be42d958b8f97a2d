"""Low-bit-KV decode attention, oracle side (§8(f) NEXT-2).  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

What the paper's attention pipeline computes (§3.4 "Attention pipeline"; §4.2 P:374-401;
§4.4): one decode step of scaled dot-product attention over a KV cache whose keys and
values are stored in low bit width and dequantised ("I2F") before use.  Plainly, for sequence b,
query head h (KV head hk = h // G, G = Hq / Hkv, grouped-query sharing) and its L_b cached tokens:

    K[t] = (kq[t] - kz[t]) * ks[t],   V[t] = (vq[t] - vz[t]) * vs[t]        (one (scale, zero) per
                                                                          token and KV head)
    S[t] = scale * sum_d Q[h][d] * K[t][d]
    P    = softmax(S) over t < L_b           (max-subtracted form, exact in float64)
    O[h] = sum_t P[t] * V[t]

computed here in float64 on exactly dequantised values (a 4-8 bit integer times an fp16 scale is
exact in float64); numpy exp and matmul are the library primitives.  The Q rearrangement and the
macro/micro-tile loading pipeline change how the kernel reaches this result, not the result.

Pinned by tests/test_oracle_attention.py: a single cached token gives O = V[0]; identical keys
give the mean of the values; a zero query gives the mean of the values; a dominant key selects
its value; adding a constant to every key's projection leaves O unchanged (shift invariance);
an exact-rational brute force (Python fractions for the dot products, mpmath-free exp via
float64) on tiny problems; the dequantisation round trip is within scale / 2.
"""

import numpy as np


def dequant_kv(q, s, z):
    """(q - z) * s per token and head: codes [..., D], s, z [...] -> float64 [..., D]."""
    return (np.asarray(q, dtype=np.float64) - np.asarray(z, dtype=np.float64)[..., None]) * \
        np.asarray(s, dtype=np.float64)[..., None]


def decode_attention_f64(Q, kq, ks, kz, vq, vs, vz, seq_lens, scale=None):
    """Q [B][Hq][D]; codes [B][Hkv][Lmax][D]; scales/zeros [B][Hkv][Lmax]; seq_lens [B]
    -> O float64 [B][Hq][D]."""
    Q = np.asarray(Q, dtype=np.float64)
    B, Hq, D = Q.shape
    Hkv = np.asarray(kq).shape[1]
    G = Hq // Hkv
    if scale is None:
        scale = 1.0 / np.sqrt(D)
    O = np.zeros((B, Hq, D))
    for b in range(B):
        L = int(seq_lens[b])
        for hk in range(Hkv):
            K = dequant_kv(kq[b, hk, :L], ks[b, hk, :L], kz[b, hk, :L])
            V = dequant_kv(vq[b, hk, :L], vs[b, hk, :L], vz[b, hk, :L])
            for h in range(hk * G, (hk + 1) * G):
                S = scale * (K @ Q[b, h])
                P = np.exp(S - S.max())
                P /= P.sum()
                O[b, h] = P @ V
    return O
