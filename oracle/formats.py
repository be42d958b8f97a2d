"""Checkpoint formats and 8-bit weights, oracle side.  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).  §8(f) NEXT-4: "W8A16 + AWQ/GPTQ checkpoint-format converters into LAYOUT v1";
the paper evaluates AWQ and GPTQ checkpoints (§5) and 4- and 8-bit weights
(§2; "comprehensive precision format support", Contribution 2).

Checkpoint formats (the public AWQ / GPTQ conventions; the paper does not restate them):
  AWQ   qweight int32 [K][N/8]: nibble i (bits 4i..4i+3) of word [k][j] holds the code of column
        8j + AWQ_ORDER[i], AWQ_ORDER = (0, 2, 4, 6, 1, 3, 5, 7); qzeros int32 [K/g][N/8] packed the
        same way along N; scales fp16 [K/g][N].
  GPTQ  qweight int32 [K/8][N]: nibble i of word [kb][n] holds the code of row 8kb + i;
        qzeros int32 [K/g][N/8]: nibble i of word [g][j] holds (zero of column 8j + i) - offset,
        offset = 1 for GPTQ-v1 checkpoints ("zeros - 1"), 0 for v2; scales fp16 [K/g][N].
        (No act-order: rows are in natural order, g_idx[k] = k // g.)
Both decode to this build's input contract (§8(a) a1): u8 codes q [K][N], fp16 zeros [K/g][N].

8-bit weights (W8A16) by bit planes: a code q8 = 16 hi + lo and zero z8 = 16 zh + zl (integers,
0..255) give  (q8 - z8) s = (hi - zh)(16 s) + (lo - zl) s  exactly, so a W8 weight [K][N] is the
W4 weight [2K][N] whose first K rows are the high planes (scale 16 s, zero zh) and last K rows the
low planes (scale s, zero zl), multiplied by the activations repeated twice along K, [A | A].
"""

import numpy as np

AWQ_ORDER = (0, 2, 4, 6, 1, 3, 5, 7)


def _nibbles(words):
    w = np.asarray(words).astype(np.int64) & 0xFFFFFFFF
    return np.stack([(w >> (4 * i)) & 0xF for i in range(8)], axis=-1).astype(np.uint8)  # [..., 8]


def awq_unpack_cols(packed, N):
    """int32 [R][N/8] packed along N in AWQ order -> uint8 [R][N]."""
    nib = _nibbles(packed)                       # [R][N/8][8]: nibble i
    out = np.empty((nib.shape[0], N), dtype=np.uint8)
    for i, col in enumerate(AWQ_ORDER):
        out[:, col::8] = nib[:, :, i]
    return out


def awq_unpack(qweight, qzeros, N):
    """-> (q uint8 [K][N], z fp16 [K/g][N])."""
    return awq_unpack_cols(qweight, N), awq_unpack_cols(qzeros, N).astype(np.float16)


def gptq_unpack(qweight, qzeros, N, zero_offset=1):
    """-> (q uint8 [K][N], z fp16 [K/g][N])."""
    nib = _nibbles(qweight)                      # [K/8][N][8]: nibble i = row 8kb + i
    q = np.transpose(nib, (0, 2, 1)).reshape(-1, N)
    zn = _nibbles(qzeros)                        # [K/g][N/8][8]: nibble i = column 8j + i
    z = zn.reshape(zn.shape[0], N).astype(np.int64) + zero_offset
    return q, z.astype(np.float16)


def awq_pack_cols(codes):
    """uint8 [R][N] -> int32 [R][N/8] (AWQ nibble order)."""
    codes = np.asarray(codes).astype(np.int64) & 0xF
    R, N = codes.shape
    w = np.zeros((R, N // 8), dtype=np.int64)
    for i, col in enumerate(AWQ_ORDER):
        w |= codes[:, col::8] << (4 * i)
    return w.astype(np.uint32).view(np.int32)


def gptq_pack(q, z, zero_offset=1):
    """(q uint8 [K][N], integer z [K/g][N]) -> (qweight int32 [K/8][N], qzeros int32 [K/g][N/8])."""
    q = np.asarray(q).astype(np.int64) & 0xF
    K, N = q.shape
    qw = np.zeros((K // 8, N), dtype=np.int64)
    for i in range(8):
        qw |= q[i::8, :] << (4 * i)
    zz = (np.asarray(z).astype(np.int64) - zero_offset) & 0xF
    qz = np.zeros((zz.shape[0], N // 8), dtype=np.int64)
    for i in range(8):
        qz |= zz[:, i::8] << (4 * i)
    return qw.astype(np.uint32).view(np.int32), qz.astype(np.uint32).view(np.int32)


def w8_bitplanes(q8, s, z8):
    """W8 (q8 uint8 [K][N], s fp16 [K/g][N], integer z8 [K/g][N]) -> W4 over 2K rows."""
    q8 = np.asarray(q8).astype(np.uint8)
    z8 = np.asarray(z8).astype(np.int64)
    q4 = np.concatenate([q8 >> 4, q8 & 15]).astype(np.uint8)
    s4 = np.concatenate([(np.asarray(s, dtype=np.float32) * 16).astype(np.float16), np.asarray(s, dtype=np.float16)])
    z4 = np.concatenate([z8 >> 4, z8 & 15]).astype(np.float16)
    return q4, s4, z4


def w8a16_gemm_f64(A, q8, s, z8, group):
    """Plain definition C[m][n] = sum_k A[m][k] (q8[k][n] - z8[k//g][n]) s[k//g][n] in float64."""
    A = np.asarray(A, dtype=np.float64)
    K, N = np.asarray(q8).shape
    z = np.repeat(np.asarray(z8, dtype=np.float64), group, axis=0)
    sc = np.repeat(np.asarray(s, dtype=np.float64), group, axis=0)
    C = np.empty((A.shape[0], N))
    for c0 in range(0, N, 4096):
        sl = slice(c0, min(N, c0 + 4096))
        C[:, sl] = A @ ((np.asarray(q8)[:, sl].astype(np.float64) - z[:, sl]) * sc[:, sl])
    return C
