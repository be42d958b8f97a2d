"""Pins for oracle/layout_v1.py (LAYOUT v1 pack / unpack).

The pins check what the layout is FOR (§4.1 P:317-326,
App. C) from the consumer's side, not by restating the pack formula:
bijection, one contiguous blob per (n-tile, k-stage), the hand-worked word, and a
simulation of the kernel's reads (LDS.128 at j*2048 + t*16, then
(w >> 4i) & 0x000F000F) that must return k-consecutive codes of row t.
"""

import json
import os

import numpy as np
import pytest

from oracle import layout_v1 as L

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("K,N", [(64, 128), (256, 256), (192, 384), (4096, 128)])
def test_roundtrip(K, N):
    rng = np.random.default_rng(K * 7 + N)
    q = rng.integers(0, 256, size=(K, N), dtype=np.uint8)  # high nibble must be ignored
    p = L.pack(q)
    assert p.dtype == np.uint8 and p.size == K * N // 2 == L.packed_bytes(K, N)
    assert np.array_equal(L.unpack(p, K, N), q & 0xF)


@pytest.mark.parametrize("K,N", [(64, 128), (128, 256)])
def test_bijection_and_blob_contiguity_by_onehot(K, N):
    """Every (k, n) lands in exactly one nibble, all nibbles are hit once, and the
    nibble lies inside the 4096-byte blob of its (n-tile, k-stage)."""
    KS = K // 64
    seen = np.zeros(K * N, dtype=np.int64)  # nibble slots
    for k in range(K):
        q = np.zeros((K, N), dtype=np.uint8)
        q[k, :] = 0xF  # one-hot row k
        p = L.pack(q).view(np.uint32)
        # decode nibble positions of row k (all columns one-hot in row k)
        nz = []
        for wi in np.nonzero(p)[0]:
            for nib in range(8):
                if (int(p[wi]) >> (4 * nib)) & 0xF:
                    nz.append(wi * 8 + nib)
        assert len(nz) == N
        for slot in nz:
            seen[slot] += 1
            byte = slot // 2
            blob = byte // 4096
            nt, ks = divmod(blob, KS)
            assert ks == k // 64
    assert np.all(seen == 1)
    # per-column check of the n-tile ownership with single one-hot elements
    rng = np.random.default_rng(3)
    for _ in range(40):
        k, n = int(rng.integers(K)), int(rng.integers(N))
        q = np.zeros((K, N), dtype=np.uint8)
        q[k, n] = 9
        p = L.pack(q)
        nzb = np.nonzero(p)[0]
        assert nzb.size == 1
        blob = nzb[0] // 4096
        assert divmod(blob, KS) == (n // 128, k // 64)


def test_loops_equal_vectorised():
    rng = np.random.default_rng(5)
    q = rng.integers(0, 16, size=(128, 256), dtype=np.uint8)
    assert np.array_equal(L.pack_loops(q.tolist()), L.pack(q))


def test_constant_codes():
    for c in (0, 1, 7, 15):
        p = L.pack(np.full((128, 256), c, dtype=np.uint8)).view(np.uint32)
        assert np.all(p == np.uint32(c * 0x11111111))


def test_hand_worked_word():
    g = json.load(open(os.path.join(GOLDEN, "layout_v1_word.json")))
    q = np.zeros((64, 128), dtype=np.uint8)
    q[0:8, 0] = g["codes"]  # thread t = 0, k = 0..7 (j = 0, wj = 0)
    w = L.pack(q).view(np.uint32)
    assert int(w[0]) == int(g["word_hex"], 16)
    pairs = [((int(w[0]) >> (4 * i)) & 0xF, (int(w[0]) >> (4 * i + 16)) & 0xF) for i in range(4)]
    assert pairs == [tuple(p) for p in g["pairs"]]


def test_consumer_simulation():
    """Simulate the dequant thread's reads of one stage and check k-consecutive order."""
    K, N = 256, 384
    rng = np.random.default_rng(11)
    q = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
    raw = L.pack(q)
    KS = K // 64
    for nt in range(N // 128):
        for ks in range(KS):
            blob = raw[(nt * KS + ks) * 4096:(nt * KS + ks + 1) * 4096]
            for t in range(128):
                got = []
                for j in range(2):
                    chunk = blob[j * 2048 + t * 16: j * 2048 + t * 16 + 16].view(np.uint32)  # LDS.128
                    for word in chunk:
                        for i in range(4):
                            v = (int(word) >> (4 * i)) & 0x000F000F
                            got += [v & 0xFFFF, v >> 16]
                assert got == list(q[ks * 64:(ks + 1) * 64, nt * 128 + t])


def test_bank_conflict_free_reads():
    """SPEC.md S:177-194 bank model: 32 lanes, 4-byte banks, 128-bit loads are served per
    quarter-warp (8 lanes x 16 B).  The dequant read address j*2048 + t*16 touches each of
    the 32 banks exactly once per quarter-warp phase, i.e. conflict degree 1 (Challenge-II,
    PAPER.md P:202-203)."""
    for j in range(2):
        for warp in range(4):
            for quarter in range(4):
                banks = []
                for lane in range(quarter * 8, quarter * 8 + 8):
                    t = warp * 32 + lane
                    addr = j * 2048 + t * 16
                    banks += [((addr + 4 * b) // 4) % 32 for b in range(4)]
                assert sorted(banks) == list(range(32))


def test_rejects_bad_shapes():
    with pytest.raises(ValueError):
        L.pack(np.zeros((60, 128), dtype=np.uint8))
    with pytest.raises(ValueError):
        L.pack(np.zeros((64, 100), dtype=np.uint8))
