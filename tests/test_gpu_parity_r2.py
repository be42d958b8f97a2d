"""GPU parity, configurations added in round 2 (VERDICT r1 "next round" item 1): fp16 and
group-64 GEMMs at every Llama-3-8B decode shape, prefill at M = 4096 / 8192 on sampled rows,
uniform-stress data at a full decode shape, the decode kernel's integer operand exhaustively,
the caller-owned workspace entry point, and the corrupted-byte negative control.

Tolerances: oracle/compare.py (reading R12); every assertion message carries both
max_ratio (bound B + half an output ulp) and max_ratio_strict (B alone).
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import compare, layout_v1
from oracle.gemm import gemm_f64
from oracle.numerics import bf16_bits, fp16_bits
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import bits16, to_dev, to_np64

pytestmark = pytest.mark.gpu

CFG1 = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]  # qkv, o, gate_up, down
RATIO_LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                         "parity_ratios.jsonl")


def _log(tag, r):
    try:
        os.makedirs(os.path.dirname(RATIO_LOG), exist_ok=True)
        with open(RATIO_LOG, "a") as f:
            f.write(json.dumps(dict(tag=str(tag), relfro=r["relfro"], max_ratio=r["max_ratio"],
                                    max_ratio_strict=r["max_ratio_strict"])) + "\n")
    except OSError:
        pass


def _run(d, act="bf16"):
    t = to_dev(d, act)
    p = api.pack_w4(t["q"], t["s"], t["z"], d["group"])
    fn = api.gemm_w4a16 if act == "bf16" else api.gemm_w4a16_f16
    C = fn(t["A"], p, t["s"], t["z"])
    torch.cuda.synchronize()
    return C, t, p


def _check(C, d, act, rows=None, tag=""):
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], d["group"], rows=rows)
    got = to_np64(C) if rows is None else to_np64(C)[rows]
    r = compare.check(got, ref, d["A"], d["q"], d["s"], d["z"], d["group"], act)
    _log(tag, r)
    assert r["ok"], (tag, compare.summary(r))
    return r


@pytest.mark.parametrize("M", [1, 16])
@pytest.mark.parametrize("N,K", CFG1)
def test_fp16_decode_cfg1_full(M, N, K):
    """fp16 activations and output at the four CFG#1 shapes (literal per-element bound)."""
    d = synth.awq_like(M, N, K, group=128, seed=2001 + M, act_dtype="fp16")
    C, _, _ = _run(d, "fp16")
    _check(C, d, "fp16", tag=("fp16", M, N, K, api.query_gemm_config(M, N, K)))


@pytest.mark.parametrize("M", [1, 16])
@pytest.mark.parametrize("N,K", CFG1)
def test_group64_decode_cfg1_full(M, N, K):
    """group 64 (CFG#4) at the four CFG#1 decode shapes, the bench's launch configuration."""
    d = synth.awq_like(M, N, K, group=64, seed=2011 + M)
    C, _, _ = _run(d)
    _check(C, d, "bf16", tag=("g64", M, N, K, api.query_gemm_config(M, N, K)))


@pytest.mark.parametrize("M", [4096, 8192])
@pytest.mark.parametrize("N,K", CFG1)
def test_prefill_large_m_sampled_rows(M, N, K):
    """CFG#2 at the bench prefill size (M = 8192) and the north-star band (M = 4096): first,
    last, m-tile boundaries and random rows against the fp64 oracle, all N."""
    d = synth.awq_like(M, N, K, group=128, seed=2021 + M // 4096)
    C, _, _ = _run(d)
    rng = np.random.default_rng(M + N)
    rows = sorted(set([0, 1, 127, 128, 255, 256, 257, M // 2, M - 257, M - 256, M - 1] +
                      rng.integers(0, M, 13).tolist()))
    _check(C, d, "bf16", rows=rows, tag=("prefill", M, N, K))


@pytest.mark.parametrize("M", [1, 16])
def test_uniform_stress_full_decode_shape(M):
    """Uniform-stress data (q, z ~ U{0..15}) at the full gate_up shape: relative Frobenius only
    (reading R12: the per-element bound is not claimed for this distribution)."""
    d = synth.uniform(M, 28672, 4096, group=128, seed=2031 + M)
    C, _, _ = _run(d)
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    rf = compare.relfro(to_np64(C), ref)
    _log(("uniform", M), dict(relfro=rf, max_ratio=float("nan"), max_ratio_strict=float("nan")))
    assert rf <= compare.RELFRO_TOL, rf


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("group", [64, 128])
def test_decode_integer_operand_exhaustive(dtype, group):
    """The decode kernel's MMA operand (reading R6b) for all 16 codes x 16 integer zeros, through
    its own deq_word_int / zero_operand code (tm_debug_dequant_int): exactly q - z, bit for bit
    (q = z gives +0)."""
    K, N = 2 * 128, 256
    q = np.tile((np.arange(K) % 16).astype(np.uint8)[:, None], (1, N))
    z = np.tile((np.arange(N) % 16).astype(np.float16)[None, :], (K // group, 1))
    s = np.ones((K // group, N), dtype=np.float16)
    dq, ds, dz = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (q, s, z))
    p = api.pack_w4(dq, ds, dz, group)
    got = bits16(api.debug_dequant_int(p, dz, dtype))
    exact = q.astype(np.float64) - np.repeat(z.astype(np.float64), group, axis=0)
    ref = bf16_bits(exact) if dtype == "bf16" else fp16_bits(exact)
    mism = np.nonzero(got != ref)
    assert mism[0].size == 0, (dtype, mism[0][:5], mism[1][:5])


def test_caller_workspace_matches_library_workspace():
    """tm_gemm_w4a16_ws with a caller-owned zero-filled workspace: bit-identical to the
    convenience entry point, leaves the workspace zeroed (flags), and refuses a missing one."""
    M, N, K = 16, 28672, 4096                       # stream-K shape: needs a workspace
    assert api.query_gemm_config(M, N, K)["kind"] == 1
    d = synth.awq_like(M, N, K, group=128, seed=2041)
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    ws = api.gemm_workspace(M, N, K, 128)
    assert ws is not None and ws.numel() == api.gemm_workspace_bytes(M, N, K, 128)
    C_ws = api.gemm_w4a16_ws(t["A"], p, t["s"], t["z"], ws)
    C_ws2 = api.gemm_w4a16_ws(t["A"], p, t["s"], t["z"], ws)
    C_lib = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    torch.cuda.synchronize()
    assert np.array_equal(bits16(C_ws), bits16(C_lib)) and np.array_equal(bits16(C_ws2), bits16(C_lib))
    P = api.query_gemm_config(M, N, K)["grid_ctas"]
    assert int(ws[:4 * P].view(torch.int32).abs().sum()) == 0   # every raised flag returned to zero
    _check(C_ws, d, "bf16", tag="workspace")
    with pytest.raises(api.TMError, match="INVALID_ARG"):
        api.gemm_w4a16_ws(t["A"], p, t["s"], t["z"], None)
    with pytest.raises(api.TMError, match="INVALID_ARG"):
        api.gemm_w4a16_ws(t["A"], p, t["s"], t["z"], ws[:64])
    # shapes routed to cluster split-K need none; fp32 partial output through the same entry
    assert api.gemm_workspace_bytes(16, 4096, 4096, 128) == 0
    d2 = synth.awq_like(16, 4096, 4096, group=128, seed=2042)
    t2 = to_dev(d2)
    p2 = api.pack_w4(t2["q"], t2["s"], t2["z"], 128)
    Cf = api.gemm_w4a16_ws(t2["A"], p2, t2["s"], t2["z"], None, out_dtype=torch.float32)
    torch.cuda.synchronize()
    _check(Cf, d2, "fp32", tag="workspace-f32")


@pytest.mark.parametrize("path", ["decode", "prefill"])
def test_negative_control_corrupted_packed_byte(path):
    """SPEC.md:604 "deliberately corrupted packed file -> exit 4 with index report": flipping one
    packed nibble (a code 0 -> 15 at a known (k, n), located with the oracle's LAYOUT v1 index
    formula) makes the parity check fail, and the reported worst element is in column n."""
    M = 8 if path == "decode" else 256
    N, K = 512, 1024
    d = synth.awq_like(M, N, K, group=128, seed=2051)
    d["q"][d["q"] == 0] = 1                            # no zero codes ...
    k0, n0 = 333, 300
    d["q"][k0, n0] = 0                                 # ... except the one we corrupt
    d["A"][:, k0] = 4.0                                # make the corrupted product stand out
    t = to_dev(d)
    p = api.pack_w4(t["q"], t["s"], t["z"], 128)
    C_ok = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    word, nib = (int(x) for x in layout_v1.word_and_nibble(k0, n0, K))
    mask = 0xF << (4 * nib)
    raw = p.data.view(torch.int32)
    raw[word] = raw[word] ^ (mask - (1 << 32) if mask >= 1 << 31 else mask)   # code 0 -> 15
    C_bad = api.gemm_w4a16(t["A"], p, t["s"], t["z"])
    torch.cuda.synchronize()
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    good = compare.check(to_np64(C_ok), ref, d["A"], d["q"], d["s"], d["z"], 128, "bf16")
    bad = compare.check(to_np64(C_bad), ref, d["A"], d["q"], d["s"], d["z"], 128, "bf16")
    assert good["ok"], compare.summary(good)
    assert not bad["ok"] and bad["argmax"][1] == n0, compare.summary(bad)
    assert np.array_equal(api.unpack_w4(p).cpu().numpy()[k0, n0], 15)
