"""GPU parity of the low-bit-KV decode attention (tm_attn_decode_kv8) against oracle/attention.py.

Tolerance (reading R18): relative Frobenius error <= 5e-3 and, per element,
|O - O_ref| <= ulp_out(O_ref) + 2e-3 * max_t |V[t]| (one output rounding plus fp32 softmax /
accumulation error; the scores see the exact dequantised keys because the codes, 1024 + code,
are exact fp16 MMA operands and Q converts exactly to fp16)."""

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.attention import decode_attention_f64, dequant_kv
from oracle.numerics import ulp
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import to_np64

pytestmark = pytest.mark.gpu


def _run(p, act="bf16"):
    tdt = torch.bfloat16 if act == "bf16" else torch.float16
    Q = torch.from_numpy(p["Q"]).to(tdt).cuda()
    kc, vc = torch.from_numpy(p["kq"]).cuda(), torch.from_numpy(p["vq"]).cuda()
    ksz = api.pack_kv_sz(torch.from_numpy(p["ks"]).cuda(), torch.from_numpy(p["kz"]).cuda())
    vsz = api.pack_kv_sz(torch.from_numpy(p["vs"]).cuda(), torch.from_numpy(p["vz"]).cuda())
    sl = torch.from_numpy(p["seq_lens"]).cuda()
    B, Hq, D = Q.shape
    _, Hkv, Lmax, _ = kc.shape
    ws = api.attn_workspace(B, Hq, Hkv, Lmax)
    O = api.attn_decode_kv8(Q, kc, vc, ksz, vsz, sl, workspace=ws)
    torch.cuda.synchronize()
    return O, ws


def _check(O, p, act="bf16", tag=""):
    ref = decode_attention_f64(p["Q"], p["kq"], p["ks"], p["kz"], p["vq"], p["vs"], p["vz"], p["seq_lens"])
    got = to_np64(O)
    vmax = np.abs(dequant_kv(p["vq"], p["vs"], p["vz"])).max()
    err = np.abs(got - ref)
    bound = ulp(ref, act) + 2e-3 * vmax
    rf = compare.relfro(got, ref)
    ratio = float((err / bound).max())
    assert np.all(np.isfinite(got)) and rf <= 5e-3 and ratio <= 1.0, (tag, rf, ratio)
    return rf, ratio


@pytest.mark.parametrize("L", [1, 5, 63, 64, 65, 130, 256, 257, 1000, 4096])
def test_context_lengths(L):
    """Single token, partial micro-/macro-tiles, exactly one split, several splits."""
    Lmax = ((L + 63) // 64) * 64
    p = synth.kv_decode_problem(2, 32, 8, 128, Lmax, [L, max(1, L // 3)], 8, seed=6000 + L)
    O, _ = _run(p)
    _check(O, p, tag=L)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("act", ["bf16", "fp16"])
def test_gqa_groups_and_dtypes(G, act):
    Hkv = 4
    p = synth.kv_decode_problem(3, Hkv * G, Hkv, 128, 768, [700, 3, 513], 8, seed=6100 + G, act_dtype=act)
    O, _ = _run(p, act)
    _check(O, p, act, tag=(G, act))


def test_workspace_left_zeroed_and_deterministic():
    p = synth.kv_decode_problem(4, 32, 8, 128, 2048, [2048, 1500, 300, 7], 8, seed=6200)
    O1, ws = _run(p)
    O2, _ = _run(p)
    assert torch.equal(O1, O2)
    assert int(ws[:4 * 4 * 8].view(torch.int32).abs().sum()) == 0
    _check(O1, p, tag="ws")


def test_many_sequences_one_split_each():
    """B x Hkv >= 2 x SMs: every (sequence, KV head) is one CTA streaming its whole context through
    the macro-tile ring (no split merge)."""
    p = synth.kv_decode_problem(40, 32, 8, 128, 640, [640 - 7 * (i % 13) for i in range(40)], 8, seed=6400)
    O, ws = _run(p)
    assert ws is None
    _check(O, p, tag="one-split")


def test_single_token_is_its_value_row():
    """one cached token -> O = dequant(v) rounded once."""
    p = synth.kv_decode_problem(1, 8, 8, 128, 64, [1], 8, seed=6300)
    O, _ = _run(p)
    V0 = dequant_kv(p["vq"][0, :, 0], p["vs"][0, :, 0], p["vz"][0, :, 0])   # [Hkv][D]
    assert np.allclose(to_np64(O)[0], V0, rtol=2 ** -8, atol=0)
