"""GPU parity of the persistent prefill kernel (gemm_pk.cuh, kind 4; M >= 1024): ragged M (the
last 192-token tile partial), both groups and activation dtypes, several tiles per CTA (the
double-buffered accumulator and the s/z box ring across tile boundaries), one-hot rows
bit-exact (reading R6: weights rounded to the operand dtype before the MMA), determinism."""

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.gemm import gemm_f64
from oracle.quant import dequant_rounded
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import to_dev, to_np64
from tests.test_gpu_parity_r2 import _log

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _pk_on():
    api.set_prefill_persistent(True)
    yield
    api.set_prefill_persistent(False)


def _gemm(d, act="bf16"):
    t = to_dev(d, act)
    p = api.pack_w4(t["q"], t["s"], t["z"], d["group"])
    C = api.gemm_w4a16(t["A"], p, t["s"], t["z"]) if act == "bf16" else api.gemm_w4a16_f16(t["A"], p, t["s"], t["z"])
    torch.cuda.synchronize()
    return C


def test_kind_is_persistent():
    for M in (1024, 2048, 8192):
        cfg = api.query_gemm_config(M, 4096, 4096)
        assert cfg["kind"] == 4 and cfg["tile_m"] == 192, cfg


@pytest.mark.parametrize("M", [1024, 1025, 1151, 1345, 2049])
@pytest.mark.parametrize("group", [64, 128])
@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_ragged_m_full_oracle(M, group, act):
    d = synth.awq_like(M, 384, 1024, group=group, seed=M + group, act_dtype=act)
    C = _gemm(d, act)
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], group)
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], group, act)
    _log(("pk", M, group, act), r)
    assert r["ok"], compare.summary(r)


def test_many_tiles_per_cta_and_odd_k():
    """N = 128 x 40 n-tiles, M = 4000 (21 m-tiles): 840 tiles, ~6 per CTA; K = 1216 (19 stages:
    a partial 8-group s/z box at g = 64)."""
    M, N, K, g = 4000, 128 * 40, 1216, 64
    d = synth.awq_like(M, N, K, group=g, seed=77)
    C = _gemm(d)
    rng = np.random.default_rng(5)
    rows = sorted(set([0, 191, 192, 383, 384, M - 193, M - 192, M - 1] + rng.integers(0, M, 24).tolist()))
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], g, rows=rows)
    r = compare.check(to_np64(C)[rows], ref, d["A"][rows], d["q"], d["s"], d["z"], g, "bf16")
    _log(("pk", "many-tiles"), r)
    assert r["ok"], compare.summary(r)


@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_onehot_rows_bit_exact(act):
    M, N, K, g = 1100, 256, 512, 128
    d = synth.uniform(1, N, K, group=g, seed=19, act_dtype=act)
    rng = np.random.default_rng(3)
    ks = rng.integers(0, K, M)
    A = np.zeros((M, K), dtype=np.float32)
    A[np.arange(M), ks] = 1.0
    d["A"] = A
    C = _gemm(d, act)
    W = dequant_rounded(d["q"], d["s"], d["z"], g, act)
    assert np.array_equal(to_np64(C), W[ks])


def test_deterministic():
    d = synth.awq_like(2048, 4096, 4096, group=128, seed=8)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    outs = [api.gemm_w4a16(t["A"], p, t["s"], t["z"]).clone() for _ in range(3)]
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
