"""GPU parity of the CTA-pair prefill kernel (gemm_2sm.cuh, kind 5: tcgen05 cta_group::2, the
default for 256-token tiles without split-K when N % 256 == 0): ragged M (the last pair tile's
token halves partial or empty), both groups and activation dtypes, K with a partial s/z box,
many pair tiles per launch, W8 bit planes (the activation ring's a_ks wrap), one-hot rows
bit-exact (reading R6), agreement with the tiled kernel, determinism, sampled rows of the
CFG#2 shapes."""

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.gemm import gemm_f64
from oracle.numerics import round_to
from oracle.quant import dequant_rounded
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import to_dev, to_np64
from tests.test_gpu_parity_r2 import _log

pytestmark = pytest.mark.gpu


def _gemm(d, act="bf16"):
    t = to_dev(d, act)
    p = api.pack_w4(t["q"], t["s"], t["z"], d["group"])
    C = api.gemm_w4a16(t["A"], p, t["s"], t["z"]) if act == "bf16" else api.gemm_w4a16_f16(t["A"], p, t["s"], t["z"])
    torch.cuda.synchronize()
    return C


def test_kind_is_pair_and_toggle():
    for M, N, K in ((1024, 4096, 4096), (8192, 28672, 4096), (2048, 6144, 4096), (4096, 4096, 14336)):
        cfg = api.query_gemm_config(M, N, K)
        assert cfg["kind"] == 5 and cfg["tile_m"] == 256 and cfg["split_k"] == 1, cfg
        assert cfg["grid_ctas"] == (N // 128) * ((M + 255) // 256)
    assert api.query_gemm_config(2048, 384, 4096)["kind"] == 0  # N % 256 != 0: tiled kernel
    api.set_prefill_pair(False)
    try:
        assert api.query_gemm_config(2048, 4096, 4096)["kind"] == 0
    finally:
        api.set_prefill_pair(True)


@pytest.mark.parametrize("M", [513, 700, 1025, 1345, 2049])
@pytest.mark.parametrize("group", [64, 128])
@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_ragged_m_full_oracle(M, group, act):
    # N = 22 n-tiles: > 64 tiles from 3 m-tiles on, so the chooser keeps split 1 (kind 5)
    d = synth.awq_like(M, 2816, 1216 if group == 64 else 1024, group=group, seed=M + group, act_dtype=act)
    assert api.query_gemm_config(M, 2816, d["A"].shape[1])["kind"] == 5
    C = _gemm(d, act)
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], group)
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], group, act)
    _log(("pair", M, group, act), r)
    assert r["ok"], compare.summary(r)


def test_many_pair_tiles_sampled_rows():
    """N = 128 x 40 (20 pairs), M = 4000 (16 m-tiles, the last 160 tokens: the peer's half
    partial), K = 1216 at g = 64 (19 stages: a partial 8-group s/z box, a ragged 4-stage flag
    group and an 11-slot activation ring wrapping mid-tile)."""
    M, N, K, g = 4000, 128 * 40, 1216, 64
    d = synth.awq_like(M, N, K, group=g, seed=78)
    C = _gemm(d)
    rng = np.random.default_rng(6)
    rows = sorted(set([0, 127, 128, 255, 256, 3839, 3840, 3967, 3968, M - 1] + rng.integers(0, M, 24).tolist()))
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], g, rows=rows)
    r = compare.check(to_np64(C)[rows], ref, d["A"][rows], d["q"], d["s"], d["z"], g, "bf16")
    _log(("pair", "many-tiles"), r)
    assert r["ok"], compare.summary(r)


@pytest.mark.parametrize("M,N,K", [(8192, 28672, 4096), (8192, 4096, 14336), (2048, 6144, 4096)])
def test_cfg2_sampled_rows(M, N, K):
    d = synth.awq_like_torch(M, N, K, seed=M + N)
    p = api.pack_w4(d["q"], d["s"], d["z"], 128)
    C = api.gemm_w4a16(d["A"], p, d["s"], d["z"])
    torch.cuda.synchronize()
    rng = np.random.default_rng(M + K)
    rows = sorted(set([0, 255, 256, M - 1] + rng.integers(0, M, 12).tolist()))
    A = d["A"].float().cpu().numpy()[rows]
    q, s, z = (d[k].cpu().numpy() for k in ("q", "s", "z"))
    ref = gemm_f64(A, q, s, z, 128)
    r = compare.check(to_np64(C)[rows], ref, A, q, s, z, 128, "bf16")
    _log(("pair-cfg2", M, N, K), r)
    assert r["ok"], compare.summary(r)


@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_onehot_rows_bit_exact(act):
    M, N, K, g = 1100, 2816, 512, 128
    d = synth.uniform(1, N, K, group=g, seed=20, act_dtype=act)
    rng = np.random.default_rng(4)
    ks = rng.integers(0, K, M)
    A = np.zeros((M, K), dtype=np.float32)
    A[np.arange(M), ks] = 1.0
    d["A"] = A
    C = _gemm(d, act)
    W = dequant_rounded(d["q"], d["s"], d["z"], g, act)
    assert np.array_equal(to_np64(C), W[ks])


@pytest.mark.parametrize("M,N,K,g", [(1024, 4096, 4096, 128), (700, 2816, 1216, 64), (2304, 1024, 2048, 128)])
def test_matches_tiled_kernel(M, N, K, g):
    """Same MMA order along K per output element as the tiled kernel (64-k stages, K = 16 per
    MMA): the two kernels agree bit for bit."""
    d = synth.awq_like(M, N, K, group=g, seed=K + g)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], g)
    C_pair = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    api.set_prefill_pair(False)
    try:
        assert api.query_gemm_config(M, N, K)["kind"] == 0
        C_tiled = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    finally:
        api.set_prefill_pair(True)
    torch.cuda.synchronize()
    assert torch.equal(C_pair, C_tiled)


def test_w8a16_bit_planes():
    """W8 (two 4-bit planes, K' = 2 K): the activation producer wraps a_ks and the low planes
    reuse the activation tiles."""
    M, N, K, g = 1024, 2816, 2048, 128
    rng = np.random.default_rng(22)
    q8 = rng.integers(0, 256, size=(K, N), dtype=np.uint8)
    z8 = rng.integers(0, 256, size=(K // g, N)).astype(np.float16)
    s = (rng.uniform(0.5, 1.0, size=(K // g, N)) * 2.0 ** -10).astype(np.float16)
    A = round_to(rng.standard_normal((M, K)), "bf16").astype(np.float32)
    dev = "cuda"
    p, s2, z2 = api.pack_w8(torch.from_numpy(q8).to(dev), torch.from_numpy(s).to(dev), torch.from_numpy(z8).to(dev), g)
    C = api.gemm_w8a16(torch.from_numpy(A).to(dev).to(torch.bfloat16), p, s2, z2)
    torch.cuda.synchronize()
    W = (q8.astype(np.float64) - np.repeat(z8.astype(np.float64), g, axis=0)) * np.repeat(s.astype(np.float64), g, axis=0)
    ref = A.astype(np.float64) @ W
    assert compare.relfro(to_np64(C), ref) <= compare.RELFRO_TOL


def test_deterministic():
    d = synth.awq_like(2048, 4096, 4096, group=128, seed=9)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    outs = [api.gemm_w4a16(t["A"], p, t["s"], t["z"]).clone() for _ in range(3)]
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("M", [700, 2049])
def test_fp32_partials_oracle_and_tiled(M):
    """fp32 partial output (row-parallel TP prefill): the 256 x 128 fp32 tile staged in the
    activation ring and stored as two 128-row boxes (the second skipped past M); within the f32
    bound of the oracle and bit-identical to the tiled kernel's partials."""
    N, K, g = 2816, 1024, 128
    d = synth.awq_like(M, N, K, group=g, seed=600 + M)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], g)
    C = api.gemm_w4a16_partial_f32(t["A"], p, t["s"], t["z"])
    api.set_prefill_pair(False)
    try:
        C_tiled = api.gemm_w4a16_partial_f32(t["A"], p, t["s"], t["z"])
    finally:
        api.set_prefill_pair(True)
    torch.cuda.synchronize()
    assert C.dtype == torch.float32 and torch.equal(C, C_tiled)
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], g)
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], g, "f32")
    _log(("pair", "f32", M), r)
    assert r["ok"], compare.summary(r)


# ---------------------------------------------------------------- split-K pairs (65 <= M <= 512)
@pytest.mark.parametrize("M", [65, 128, 200, 256, 300, 512])
@pytest.mark.parametrize("N,K,g", [(1024, 1216, 64), (1536, 2048, 128)])
@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_split_k_full_oracle(M, N, K, g, act):
    """Mid M: S = 4 splits of one CTA pair per cluster (2 S = 8 CTAs), each split's K range
    (K = 1216: 19 stages -> 4/5/5/5, s/z boxes straddling the split points at g = 64), the
    token slices exchanged with st.async and summed in split order; ragged M (65, 200, 300:
    chunks past M neither sent nor stored)."""
    cfg = api.query_gemm_config(M, N, K)
    assert cfg["kind"] == 5 and cfg["split_k"] > 1, cfg
    d = synth.awq_like(M, N, K, group=g, seed=M * 7 + N + g, act_dtype=act)
    C = _gemm(d, act)
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], g)
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], g, act)
    _log(("pair-split", M, N, K, act), r)
    assert r["ok"], compare.summary(r)


@pytest.mark.parametrize("M,N,K", [(256, 6144, 4096), (128, 4096, 14336), (512, 4096, 4096), (100, 4096, 4096)])
def test_split_k_cfg_shapes_sampled_rows(M, N, K):
    cfg = api.query_gemm_config(M, N, K)
    assert cfg["kind"] == 5 and cfg["split_k"] > 1, cfg
    d = synth.awq_like_torch(M, N, K, seed=M + N + K)
    p = api.pack_w4(d["q"], d["s"], d["z"], 128)
    C = api.gemm_w4a16(d["A"], p, d["s"], d["z"])
    torch.cuda.synchronize()
    rng = np.random.default_rng(M)
    rows = sorted(set([0, M // 2, M - 1] + rng.integers(0, M, 9).tolist()))
    A = d["A"].float().cpu().numpy()[rows]
    q, s, z = (d[k].cpu().numpy() for k in ("q", "s", "z"))
    ref = gemm_f64(A, q, s, z, 128)
    r = compare.check(to_np64(C)[rows], ref, A, q, s, z, 128, "bf16")
    _log(("pair-split-cfg", M, N, K), r)
    assert r["ok"], compare.summary(r)


def test_split_k_fp32_partials_and_determinism():
    M, N, K, g = 256, 1536, 2048, 128
    d = synth.awq_like(M, N, K, group=g, seed=31)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], g)
    outs = [api.gemm_w4a16_partial_f32(t["A"], p, t["s"], t["z"]).clone() for _ in range(3)]
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], g)
    r = compare.check(to_np64(outs[0]), ref, d["A"], d["q"], d["s"], d["z"], g, "f32")
    _log(("pair-split", "f32"), r)
    assert r["ok"], compare.summary(r)


def test_split_k_w8_bit_planes():
    M, N, K, g = 256, 2816, 2048, 128
    assert api.query_gemm_config(M, N, 2 * K)["split_k"] > 1
    rng = np.random.default_rng(23)
    q8 = rng.integers(0, 256, size=(K, N), dtype=np.uint8)
    z8 = rng.integers(0, 256, size=(K // g, N)).astype(np.float16)
    s = (rng.uniform(0.5, 1.0, size=(K // g, N)) * 2.0 ** -10).astype(np.float16)
    A = round_to(rng.standard_normal((M, K)), "bf16").astype(np.float32)
    dev = "cuda"
    p, s2, z2 = api.pack_w8(torch.from_numpy(q8).to(dev), torch.from_numpy(s).to(dev), torch.from_numpy(z8).to(dev), g)
    C = api.gemm_w8a16(torch.from_numpy(A).to(dev).to(torch.bfloat16), p, s2, z2)
    torch.cuda.synchronize()
    W = (q8.astype(np.float64) - np.repeat(z8.astype(np.float64), g, axis=0)) * np.repeat(s.astype(np.float64), g, axis=0)
    assert compare.relfro(to_np64(C), A.astype(np.float64) @ W) <= compare.RELFRO_TOL


# ---------------------------------------------------------------- 64-token pair tiles (opt-in)
@pytest.mark.parametrize("M,N,K,g", [(64, 1024, 1216, 64), (17, 2816, 2048, 128), (40, 1536, 2048, 128)])
@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_pair64_opt_in_full_oracle(M, N, K, g, act):
    """tm_set_prefill_pair(2): 17 <= M <= 64 on 64-token pair tiles (M = 256 x N = 64 MMAs, each
    CTA staging 32 tokens), split-K over the cluster with 16-token slices (4 chunks per tile)."""
    api.set_prefill_pair(2)
    try:
        cfg = api.query_gemm_config(M, N, K)
        assert cfg["kind"] == 5 and cfg["tile_m"] == 64 and cfg["split_k"] > 1, cfg
        d = synth.awq_like(M, N, K, group=g, seed=M * 3 + N + g, act_dtype=act)
        C = _gemm(d, act)
    finally:
        api.set_prefill_pair(True)
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], g)
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], g, act)
    _log(("pair64", M, N, K, act), r)
    assert r["ok"], compare.summary(r)


def test_set_prefill_pair_rejects_bad_mode():
    with pytest.raises(api.TMError):
        api.set_prefill_pair(4)


def test_mid_m_128_token_tiles_and_mode3():
    """M <= 128 runs 128-token pair tiles (default); mode 3 keeps 256-token tiles there (A/B)."""
    assert api.query_gemm_config(128, 4096, 4096)["tile_m"] == 128
    api.set_prefill_pair(3)
    try:
        assert api.query_gemm_config(128, 4096, 4096)["tile_m"] == 256
    finally:
        api.set_prefill_pair(True)
