"""LAYOUT v1: the offline packing of u4 weight codes (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What the paper fixes (§4.1 "Hardware-aware weight packing steps",
P:317-326, and App. C): the packed format is chosen offline so that the
online kernel loads a tile with one coalesced copy, reads it from shared memory
without bank conflicts, and finds the sub-word values already in the order the
dequantiser/MMA wants ("permuting the sub-word values into the exact order
expected by the MMA instruction").  The concrete Ampere format (Figs 6-8)
is prior art and its figures are not recoverable ([FIGURE]), so the
build defines its own sm_100a format, LAYOUT v1 (reading R10).
This module is that definition written out as a plain index formula:

  tile BN = 128 weight columns n (one per TMEM lane / dequant thread),
  stage BK = 64 reduction indices k (one TMA bulk copy of 4096 bytes).

  For element (k, n) of q[K][N]:
      t  = n % 128         nt = n // 128
      ks = k // 64         kk = k % 64
      w  = kk // 8         j  = w // 4        wj = w % 4        e = kk % 8
      word   = ((nt * (K // 64) + ks) * 2 + j) * 512 + t * 4 + wj
      nibble = (e % 2) * 4 + e // 2            (bits [4*nibble, 4*nibble+4) of the
                                                little-endian 32-bit word)

So a word holds k-consecutive codes [e0 e2 e4 e6 e1 e3 e5 e7] in nibbles 0..7,
(w >> 4i) & 0x000F000F yields the pair (e_{2i}, e_{2i+1}) in the two 16-bit
halves, thread t's 16 bytes at blob offset j*2048 + t*16 are 32 k-consecutive
codes of its row, and every (nt, ks) stage is one contiguous 4096-byte blob.

Pinned by tests/test_oracle_layout.py: round trip, bijection by one-hot
enumeration, blob contiguity, constant codes, the hand-worked word 0x86427531,
and a consumer simulation written from the reader's side (LDS.128 + LOP3 pairs)
rather than from this formula.
"""

import numpy as np

BN = 128
BK = 64


def check_shape(K, N):
    if K <= 0 or N <= 0 or K % BK or N % BN:
        raise ValueError(f"LAYOUT v1 needs K % {BK} == 0 and N % {BN} == 0, got K={K} N={N}")


def packed_bytes(K, N):
    check_shape(K, N)
    return K * N // 2


def word_and_nibble(k, n, K):
    """Vectorised formula: (word index, nibble index) for element (k, n)."""
    k = np.asarray(k, dtype=np.int64)
    n = np.asarray(n, dtype=np.int64)
    t, nt = n % BN, n // BN
    ks, kk = k // BK, k % BK
    w = kk // 8
    j, wj, e = w // 4, w % 4, kk % 8
    word = ((nt * (K // BK) + ks) * 2 + j) * 512 + t * 4 + wj
    nib = (e % 2) * 4 + e // 2
    return word, nib


def pack(q):
    """q: uint8 [K][N] codes (only the low nibble is used) -> uint8 [K*N/2] packed bytes.

    Walks one 128-column n-tile at a time only to bound memory; each element is
    placed by word_and_nibble() above, nothing else."""
    q = np.asarray(q)
    K, N = q.shape
    check_shape(K, N)
    words = np.zeros(K * N // 8, dtype=np.uint32)
    kk, tt = np.meshgrid(np.arange(K), np.arange(BN), indexing="ij")
    for nt in range(N // BN):
        codes = q[:, nt * BN:(nt + 1) * BN].astype(np.uint32) & 0xF
        word, nib = word_and_nibble(kk, tt + nt * BN, K)
        # each (word, nibble) slot is written exactly once (bijection), so OR == assignment
        np.bitwise_or.at(words, word.ravel(), (codes << (4 * nib.astype(np.uint32))).ravel())
    return words.view(np.uint8).copy()


def unpack(packed, K, N):
    """Inverse of pack: uint8 [K*N/2] -> uint8 [K][N] codes in 0..15."""
    check_shape(K, N)
    words = np.ascontiguousarray(packed, dtype=np.uint8).view(np.uint32)
    if words.size != K * N // 8:
        raise ValueError("packed size does not match K, N")
    q = np.empty((K, N), dtype=np.uint8)
    kk, tt = np.meshgrid(np.arange(K), np.arange(BN), indexing="ij")
    for nt in range(N // BN):
        word, nib = word_and_nibble(kk, tt + nt * BN, K)
        q[:, nt * BN:(nt + 1) * BN] = (words[word] >> (4 * nib.astype(np.uint32))) & 0xF
    return q


def pack_loops(q):
    """Pure-Python element-at-a-time pack of the same formula (tiny shapes only)."""
    K, N = len(q), len(q[0])
    check_shape(K, N)
    words = [0] * (K * N // 8)
    for k in range(K):
        for n in range(N):
            t, nt = n % BN, n // BN
            ks, kk = k // BK, k % BK
            w = kk // 8
            j, wj, e = w // 4, w % 4, kk % 8
            word = ((nt * (K // BK) + ks) * 2 + j) * 512 + t * 4 + wj
            nib = (e % 2) * 4 + e // 2
            words[word] |= (int(q[k][n]) & 0xF) << (4 * nib)
    return np.array(words, dtype=np.uint32).view(np.uint8)
