"""GPU parity: tm_gemm_w4a16 (+ _f16, _partial_f32) against the fp64 oracle.

Tolerances (north star; DESIGN.md §4 R12): relative Frobenius error <= 5e-3 and the
per-element bound of oracle/compare.py; closed forms are bit-exact.
"""

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.gemm import gemm_f64
from oracle.quant import dequant_rounded, dequant_f64
from oracle.numerics import round_to
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import to_dev, to_np64, bits16
from tests.test_gpu_parity_r2 import _log

pytestmark = pytest.mark.gpu

TILES = [(16, 1), (16, 2), (16, 4), (16, 8), (32, 3), (64, 2), (128, 1), (256, 1), (64, 1), (128, 2)]


@pytest.fixture(autouse=True)
def _reset_override():
    api.set_gemm_override(0, 0)
    yield
    api.set_gemm_override(0, 0)


def _run(d, act="bf16", out="act"):
    t = to_dev(d, act)
    p = api.pack_w4(t["q"], t["s"], t["z"], d["group"])
    if out == "f32":
        C = api.gemm_w4a16_partial_f32(t["A"], p, t["s"], t["z"])
    elif act == "bf16":
        C = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    else:
        C = api.gemm_w4a16_f16(t["A"], p, t["s"], t["z"])
    torch.cuda.synchronize()
    return C, t, p


def _assert_parity(C, d, act="bf16", rows=None, tag=""):
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], d["group"], rows=rows)
    got = to_np64(C) if rows is None else to_np64(C)[rows]
    r = compare.check(got, ref, d["A"], d["q"], d["s"], d["z"], d["group"], act)
    _log(tag, r)
    assert r["ok"], (tag, compare.summary(r))
    return r


@pytest.mark.parametrize("act", ["bf16", "fp16"])
@pytest.mark.parametrize("kind", ["awq", "uniform"])
def test_tiny_config(act, kind):
    """CFG#0: M=4 N=256 K=256 group=128."""
    gen = synth.awq_like if kind == "awq" else synth.uniform
    d = gen(4, 256, 256, group=128, seed=1000 if kind == "awq" else 1001, act_dtype=act)
    C, _, _ = _run(d, act)
    if kind == "awq":
        _assert_parity(C, d, act)
    else:  # uniform stress: relFro only (reading R12)
        ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
        assert compare.relfro(to_np64(C), ref) <= compare.RELFRO_TOL


@pytest.mark.parametrize("tile,split", TILES)
@pytest.mark.parametrize("group", [64, 128])
def test_every_variant_ragged(tile, split, group):
    """Every (tile_m, split-K) variant on a shape spanning several tiles with ragged M."""
    api.set_gemm_override(tile, split)
    for M in (1, 3, tile - 1 if tile > 1 else 1, tile + 5, 2 * tile + 1):
        d = synth.awq_like(M, 384, 1024, group=group, seed=M * 31 + tile + split)
        C, _, _ = _run(d)
        _assert_parity(C, d, tag=(tile, split, M))


@pytest.mark.parametrize("M", [1, 2, 3, 5, 7, 8, 9, 15, 16, 17, 31, 33, 63, 65, 127, 129, 255, 257])
def test_auto_config_ragged_M(M):
    d = synth.awq_like(M, 512, 768, group=128, seed=100 + M)
    C, _, _ = _run(d)
    _assert_parity(C, d, tag=M)


@pytest.mark.parametrize("M", [1, 8, 16])
@pytest.mark.parametrize("N,K", [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)])
def test_llama3_8b_decode_full(M, N, K):
    """CFG#1 at full size, bench launch configuration, full fp64 oracle."""
    d = synth.awq_like(M, N, K, group=128, seed=1001)
    C, _, _ = _run(d)
    _assert_parity(C, d, tag=(M, N, K))


@pytest.mark.parametrize("M", [1, 16])
@pytest.mark.parametrize("N,K", [(57344, 8192), (8192, 28672), (59136, 8192), (8192, 29568)])
def test_70b_qwen72b_decode_full(M, N, K):
    """CFG#3/CFG#4 decode shapes at full size (Llama-3-70B gate_up/down, Qwen2-72B gate_up/down;
    Qwen2-72B down K=29568 ends in a half chunk: the K-tail path at scale), full fp64 oracle."""
    d = synth.awq_like(M, N, K, group=128, seed=1005 + M)
    C, _, _ = _run(d)
    _assert_parity(C, d, tag=(M, N, K, api.query_gemm_config(M, N, K)))


@pytest.mark.parametrize("M", [100, 128, 200, 256, 512])
@pytest.mark.parametrize("N,K", [(6144, 4096), (4096, 4096), (4096, 14336)])
def test_llama3_8b_mid_m_split_configs(M, N, K):
    """Mid M (65..512): the auto configuration splits K over a cluster of 2-4 CTAs per tile
    (api.cu choose_config); full fp64 oracle on every row."""
    cfg = api.query_gemm_config(M, N, K)
    d = synth.awq_like(M, N, K, group=128, seed=1003 + M)
    C, _, _ = _run(d)
    _assert_parity(C, d, tag=(M, N, K, cfg))


@pytest.mark.parametrize("N,K", [(6144, 4096), (28672, 4096), (4096, 14336)])
def test_llama3_8b_prefill_sampled_rows(N, K):
    """CFG#2 (M=2048): sampled rows (first, last, tile boundaries, random) vs the oracle."""
    M = 2048
    d = synth.awq_like(M, N, K, group=128, seed=1002)
    C, _, _ = _run(d)
    rng = np.random.default_rng(0)
    rows = sorted(set([0, 1, 255, 256, 257, 1023, 1024, M - 1] + rng.integers(0, M, 24).tolist()))
    _assert_parity(C, d, rows=rows, tag=(N, K))


@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_zero_weights_exact(act):
    rng = np.random.default_rng(1)
    K, N, g = 512, 384, 128
    z = rng.integers(0, 16, size=(K // g, N)).astype(np.float16)
    q = np.repeat(z.astype(np.uint8), g, axis=0)
    s = rng.uniform(0.001, 0.1, size=(K // g, N)).astype(np.float16)
    d = dict(A=synth.round_act(rng.normal(size=(20, K)), act), q=q, s=s, z=z, group=g, act_dtype=act)
    C, _, _ = _run(d, act)
    assert torch.all(C == 0)


@pytest.mark.parametrize("act", ["bf16", "fp16"])
@pytest.mark.parametrize("path", ["decode", "tiled"])
def test_onehot_rows_are_dequant_rows_bit_exact(act, path):
    """A one-hot activation row selects one dequantised weight row.  Decode path (reading
    R6b: exact (q - z) operand, scale in fp32, one output rounding): RNE((q - z) * s).
    Tiled path (reading R6: weights rounded to the operand dtype before the MMA): the
    rounding sequence of oracle.quant.dequant_rounded."""
    d = synth.uniform(1, 384, 512, group=128, seed=9, act_dtype=act)
    ks = [0, 1, 63, 64, 127, 128, 300, 511]
    A = np.zeros((len(ks), 512), dtype=np.float32)
    for m, k in enumerate(ks):
        A[m, k] = 1.0
    d["A"] = A
    if path == "tiled":
        api.set_gemm_override(128, 1)
    C, _, _ = _run(d, act)
    if path == "decode":
        W = round_to(dequant_f64(d["q"], d["s"], d["z"], 128), act)
    else:
        W = dequant_rounded(d["q"], d["s"], d["z"], 128, act)
    assert np.array_equal(to_np64(C), W[ks])


def test_ones_activation_power_of_two_scales_bit_exact():
    rng = np.random.default_rng(12)
    K, N, g = 1024, 256, 128
    q = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
    z = rng.integers(0, 16, size=(K // g, N)).astype(np.float16)
    s = np.full((K // g, N), 2.0 ** -5, dtype=np.float16)
    d = dict(A=np.ones((3, K), dtype=np.float32), q=q, s=s, z=z, group=g, act_dtype="bf16")
    C, _, _ = _run(d)
    exact = gemm_f64(d["A"], q, s, z, g)
    assert np.array_equal(to_np64(C), round_to(exact, "bf16"))


def test_doubling_activation_doubles_output():
    d = synth.awq_like(9, 256, 512, seed=21)
    C1, _, _ = _run(d)
    d2 = dict(d, A=d["A"] * 2.0)
    C2, _, _ = _run(d2)
    assert torch.equal(C2.float(), 2.0 * C1.float())


def test_deterministic_run_to_run():
    d = synth.awq_like(16, 1024, 4096, seed=33)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    outs = [bits16(api.gemm_w4a16(t["A"], p, t["s"], t["z"])) for _ in range(3)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_partial_f32_and_finalize():
    d = synth.awq_like(16, 512, 2048, seed=44)
    C, t, p = _run(d, out="f32")
    assert C.dtype == torch.float32
    _assert_parity(C, d, act="fp32")
    Cb = api.tp_finalize(C)
    assert torch.equal(Cb, C.to(torch.bfloat16))
    api.set_gemm_override(16, 1)
    Cf = api.gemm_w4a16_partial_f32(t["A"], p, t["s"], t["z"])
    Cbf = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    assert torch.equal(Cf.to(torch.bfloat16), Cbf)


def test_n_shard_concatenation_bit_exact():
    """Column-parallel TP (§8(e)): packing column shards and running them separately gives the
    same bits as the full GEMM when the launch configuration is held fixed."""
    d = synth.awq_like(16, 1024, 1024, seed=55)
    api.set_gemm_override(16, 2)
    C, t, _ = _run(d)
    parts = []
    for r in range(4):
        cols = slice(r * 256, (r + 1) * 256)
        qs, ss, zs = (x[:, cols].contiguous() for x in (t["q"], t["s"], t["z"]))
        ps = api.pack_w4(qs, ss, zs, 128)
        parts.append(api.gemm_w4a16(t["A"], ps, ss, zs))
    assert torch.equal(torch.cat(parts, dim=1), C)


def test_k_shard_partials_sum():
    """Row-parallel TP: sum of fp32 partials over K shards matches the oracle."""
    d = synth.awq_like(8, 512, 4096, seed=66)
    t = to_dev(d)
    acc = None
    for r in range(4):
        ks = slice(r * 1024, (r + 1) * 1024)
        gs = slice(r * 8, (r + 1) * 8)
        qs, ss, zs = t["q"][ks].contiguous(), t["s"][gs].contiguous(), t["z"][gs].contiguous()
        ps = api.pack_w4(qs, ss, zs, 128)
        part = api.gemm_w4a16_partial_f32(t["A"][:, ks].contiguous(), ps, ss, zs)
        acc = part if acc is None else acc + part
    _assert_parity(api.tp_finalize(acc), d)


def test_m_zero_is_noop_and_errors():
    d = synth.awq_like(1, 256, 256, seed=1)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    out = torch.full((0, 256), 7, dtype=torch.bfloat16, device="cuda")
    api.gemm_w4a16(t["A"][:0], p, t["s"], t["z"], out=out)
    bad = api.PackedW4(p.data, 256, 256, 128)  # descriptor never filled by tm_pack_w4
    with pytest.raises(api.TMError, match="INVALID_ARG"):
        api.gemm_w4a16(t["A"], bad, t["s"], t["z"])


SK_CASES = [(16, 1), (16, 3), (16, 7), (16, 148), (32, 5), (64, 4), (64, 148), (16, 2000)]


@pytest.mark.parametrize("tile,P", SK_CASES)
@pytest.mark.parametrize("group", [64, 128])
def test_streamk_variants_ragged(tile, P, group):
    """Persistent stream-K kernel with forced CTA counts P (partial tiles at every range
    boundary), ragged M, and K not a multiple of the 256-k chunk (partial last chunk)."""
    api.set_gemm_override(tile, -P)
    for M, N, K in ((1, 384, 896), (tile, 256, 1024), (tile + 3, 512, 640), (2 * tile + 1, 384, 1408)):
        d = synth.awq_like(M, N, K, group=group, seed=M * 7 + N + K + P)
        C, _, _ = _run(d)
        _assert_parity(C, d, tag=(tile, P, M, N, K))


def test_streamk_partial_f32_and_fp16():
    api.set_gemm_override(16, -5)
    d = synth.awq_like(9, 384, 1024, seed=77)
    C, _, _ = _run(d, out="f32")
    _assert_parity(C, d, act="fp32")
    d16 = synth.awq_like(9, 384, 1024, seed=78, act_dtype="fp16")
    C16, _, _ = _run(d16, act="fp16")
    _assert_parity(C16, d16, act="fp16")


def test_streamk_deterministic_and_counter_reset():
    """Repeated launches (counters must return to zero) give identical bits."""
    api.set_gemm_override(16, -37)
    d = synth.awq_like(16, 2048, 4096, seed=88)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    outs = [bits16(api.gemm_w4a16(t["A"], p, t["s"], t["z"])) for _ in range(4)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    _assert_parity(api.gemm_w4a16(t["A"], p, t["s"], t["z"]), d)


CLUSTER_CASES = [2, 3, 4, 5, 8]


@pytest.mark.parametrize("cs", CLUSTER_CASES)
@pytest.mark.parametrize("group", [64, 128])
def test_decode_cluster_split_ragged(cs, group):
    """Decode kernel in cluster mode (cs CTAs per tile, DSMEM reduction in rank order):
    ragged M (all three tile sizes), K tails, cs capped by K and by the leader's SMEM."""
    api.set_gemm_override(0, 0)
    api.set_decode_cluster(cs)
    try:
        for M, N, K in ((1, 384, 896), (16, 256, 2048), (19, 512, 640), (33, 384, 1408), (64, 256, 4096)):
            d = synth.awq_like(M, N, K, group=group, seed=M * 11 + N + K + cs)
            cfg = api.query_gemm_config(M, N, K)
            assert cfg["kind"] == 2 and 2 <= cfg["split_k"] <= cs, cfg
            C, _, _ = _run(d)
            _assert_parity(C, d, tag=(cs, M, N, K))
    finally:
        api.set_decode_cluster(0)


@pytest.mark.parametrize("group", [64, 128])
def test_decode_one_cta_per_tile_ragged(group):
    """Decode kernel with one CTA per tile and no split (forced; chosen automatically when
    70-100 % of the SMs get a whole tile): all three tile sizes, ragged M, K tails."""
    api.set_decode_cluster(-1)
    try:
        for M, N, K in ((1, 384, 896), (16, 256, 2048), (19, 512, 640), (33, 384, 1408), (64, 256, 4096)):
            d = synth.awq_like(M, N, K, group=group, seed=M * 13 + N + K)
            cfg = api.query_gemm_config(M, N, K)
            assert cfg["kind"] == 2 and cfg["split_k"] == 1, cfg
            C, _, _ = _run(d)
            _assert_parity(C, d, tag=(M, N, K))
    finally:
        api.set_decode_cluster(0)


@pytest.mark.parametrize("M", [1, 16, 40, 64])
def test_mixtral_expert_auto_one_cta_per_tile(M):
    """Mixtral expert (N=14336, K=4096; 112 tiles): the automatic choice is one CTA per tile."""
    d = synth.awq_like(M, 14336, 4096, group=128, seed=1004 + M)
    cfg = api.query_gemm_config(M, 14336, 4096)
    assert cfg["kind"] == 2 and cfg["split_k"] == 1, cfg
    C, _, _ = _run(d)
    _assert_parity(C, d, tag=(M, cfg))


def test_decode_cluster_auto_shapes_and_determinism():
    """Automatic choice on Llama-3-8B o_proj / qkv (cluster mode) is bit-stable run to run and
    within tolerance; partial f32 and fp16 variants."""
    api.set_gemm_override(0, 0)
    api.set_decode_cluster(0)
    for (M, N, K) in ((16, 4096, 4096), (8, 6144, 4096)):
        assert api.query_gemm_config(M, N, K)["kind"] == 2
        d = synth.awq_like(M, N, K, seed=N + M)
        t = to_dev(d)
        p = api.pack_w4(t["q"], t["s"], t["z"], 128)
        outs = [bits16(api.gemm_w4a16(t["A"], p, t["s"], t["z"])) for _ in range(3)]
        assert all(np.array_equal(outs[0], o) for o in outs[1:])
        _assert_parity(api.gemm_w4a16(t["A"], p, t["s"], t["z"]), d)
    d = synth.awq_like(9, 1024, 1024, seed=79)
    C, _, _ = _run(d, out="f32")
    _assert_parity(C, d, act="fp32")
    d16 = synth.awq_like(9, 1024, 1024, seed=80, act_dtype="fp16")
    C16, _, _ = _run(d16, act="fp16")
    _assert_parity(C16, d16, act="fp16")
