"""GPU parity of the register-fed decode kernel (gemm_rf.cuh, kind 3; M <= 16) against the fp64
oracle: every forced split, both groups and activation dtypes, the fp32-partial output, K tails,
ragged M, full CFG#1 shapes, determinism, the closed forms, and the W8 bit-plane path.

Reading R6c: the operand is the exact V + q, the zero point is folded back with the
activation sums, one output rounding -- tolerance-checked (R12), closed forms bit-exact.
"""

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.gemm import gemm_f64
from oracle.numerics import round_to
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import to_dev, to_np64
from tests.test_gpu_parity_r2 import _log

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _rf_path():
    api.set_gemm_override(0, 0)
    api.set_decode_cluster(0)
    api.set_decode_path(2, 0)
    yield
    api.set_decode_path(0, 0)


def _gemm(d, act="bf16", out="act"):
    t = to_dev(d, act)
    p = api.pack_w4(t["q"], t["s"], t["z"], d["group"])
    if out == "f32":
        C = api.gemm_w4a16_partial_f32(t["A"], p, t["s"], t["z"])
    elif act == "bf16":
        C = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    else:
        C = api.gemm_w4a16_f16(t["A"], p, t["s"], t["z"])
    torch.cuda.synchronize()
    return C


def _check(C, d, act="bf16", tag=""):
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], d["group"])
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], d["group"], act)
    _log(("rf",) + tuple(tag) if isinstance(tag, tuple) else ("rf", tag), r)
    assert r["ok"], (tag, compare.summary(r))
    return r


def test_kind_is_register_fed():
    for M in (1, 8, 9, 16):
        cfg = api.query_gemm_config(M, 4096, 4096)
        assert cfg["kind"] == 3 and cfg["tile_m"] == (8 if M <= 8 else 16), cfg
        assert cfg["split_k"] >= 2, cfg  # 32 tiles: cluster split
        cfg = api.query_gemm_config(M, 28672, 4096)
        assert cfg["kind"] == 3 and cfg["split_k"] < 0, cfg  # 224 tiles: stream-K
    assert api.query_gemm_config(17, 4096, 4096)["kind"] != 3


@pytest.mark.parametrize("split", [1, 2, 3, 4, 5, 8, -1, -2, -3, -7, -11, -15])
@pytest.mark.parametrize("group", [64, 128])
def test_forced_splits_ragged(split, group):
    """Several tiles, K = 1216 at g = 64 (4 full chunks + a 3-blob tail) / 1280 at g = 128 (a
    2-blob tail), every cluster split (split > 0: CTAs per tile) and stream-K CTA counts
    (split < 0: segments crossing tiles, 1..3 contributors per tile, whole and partial tiles
    mixed), ragged M on both tile sizes."""
    K = 1216 if group == 64 else 1280
    api.set_decode_path(2, split)
    for M in (1, 3, 8, 9, 13, 16):
        d = synth.awq_like(M, 384, K, group=group, seed=M * 7 + split + group)
        _check(_gemm(d), d, tag=(split, group, M))


@pytest.mark.parametrize("act", ["bf16", "fp16"])
@pytest.mark.parametrize("group", [64, 128])
@pytest.mark.parametrize("M", [1, 8, 16])
def test_dtypes_and_groups(act, group, M):
    d = synth.awq_like(M, 1024, 2048, group=group, seed=300 + M + group, act_dtype=act)
    _check(_gemm(d, act), d, act, tag=(act, group, M))


@pytest.mark.parametrize("M", [1, 5, 16])
def test_fp32_partial_output(M):
    d = synth.awq_like(M, 512, 4096, group=128, seed=400 + M)
    C = _gemm(d, out="f32")
    assert C.dtype == torch.float32
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], 128, "f32")
    _log(("rf", "f32", M), r)
    assert r["ok"], compare.summary(r)


def test_stream_k_workspace_abi():
    """Stream-K mode needs the caller workspace tm_gemm_workspace_bytes reports; the _ws entry
    point with exactly that buffer gives the library-workspace result bit for bit."""
    M, N, K = 16, 28672, 4096
    need = api.lib().tm_gemm_workspace_bytes(M, N, K, 128)
    assert need > 0
    d = synth.awq_like(M, N, K, group=128, seed=11)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    C0 = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    C1 = torch.empty_like(C0)
    api.gemm_w4a16_ws(t["A"], p, t["s"], t["z"], ws, out=C1)
    torch.cuda.synchronize()
    assert torch.equal(C0, C1)


@pytest.mark.parametrize("M", [1, 8, 16])
@pytest.mark.parametrize("N,K", [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)])
@pytest.mark.parametrize("group", [64, 128])
def test_llama3_8b_full(M, N, K, group):
    """CFG#1 at full size in the automatic launch configuration (the bench's), full oracle."""
    d = synth.awq_like(M, N, K, group=group, seed=1001)
    _check(_gemm(d), d, tag=(M, N, K, group, api.query_gemm_config(M, N, K)["split_k"]))


def test_uniform_stress_full_shape():
    """Uniform codes/zeros/scales (large |q - z|, the largest cancellation in the zero-point fold):
    relFro at a full decode shape."""
    d = synth.uniform(16, 4096, 4096, group=128, seed=77)
    C = _gemm(d)
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    assert compare.relfro(to_np64(C), ref) <= compare.RELFRO_TOL


def test_deterministic():
    d = synth.awq_like(16, 4096, 14336, group=128, seed=5)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    outs = [api.gemm_w4a16(t["A"], p, t["s"], t["z"]).clone() for _ in range(3)]
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_one_hot_closed_form(act):
    """A = e_k rows: C[m][n] = RNE((q[k_m][n] - z) * s) exactly (one product, one rounding)."""
    M, N, K, g = 16, 256, 1024, 128
    rng = np.random.default_rng(9)
    q = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
    z = rng.integers(0, 16, size=(K // g, N)).astype(np.float16)
    s = (rng.uniform(0.5, 1.0, size=(K // g, N)) * 2.0 ** -4).astype(np.float16)
    ks = rng.choice(K, size=M, replace=False)
    A = np.zeros((M, K), dtype=np.float32)
    A[np.arange(M), ks] = 1.0
    d = dict(A=A, q=q, s=s, z=z, group=g)
    C = to_np64(_gemm(d, act))
    exact = (q[ks, :].astype(np.float64) - z[ks // g, :].astype(np.float64)) * s[ks // g, :].astype(np.float64)
    assert np.array_equal(C, round_to(exact, act))


def test_w8a16_bit_planes():
    """W8 through the bit planes (A reused by the low planes): the kernel's a_ks wrap."""
    M, N, K, g = 16, 512, 2048, 128
    rng = np.random.default_rng(21)
    q8 = rng.integers(0, 256, size=(K, N), dtype=np.uint8)
    z8 = rng.integers(0, 256, size=(K // g, N)).astype(np.float16)
    s = (rng.uniform(0.5, 1.0, size=(K // g, N)) * 2.0 ** -10).astype(np.float16)
    A = rng.standard_normal((M, K)).astype(np.float32)
    A = round_to(A.astype(np.float64), "bf16").astype(np.float32)
    dev = "cuda"
    p, s2, z2 = api.pack_w8(torch.from_numpy(q8).to(dev), torch.from_numpy(s).to(dev), torch.from_numpy(z8).to(dev), g)
    C = api.gemm_w8a16(torch.from_numpy(A).to(dev).to(torch.bfloat16), p, s2, z2)
    torch.cuda.synchronize()
    W = (q8.astype(np.float64) - np.repeat(z8.astype(np.float64), g, axis=0)) * np.repeat(s.astype(np.float64), g, axis=0)
    ref = A.astype(np.float64) @ W
    assert compare.relfro(to_np64(C), ref) <= compare.RELFRO_TOL

