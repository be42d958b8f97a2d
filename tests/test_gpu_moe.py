"""GPU parity of the grouped (MoE) launch tm_gemm_w4a16_grouped against oracle/moe.py."""

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.moe import grouped_gemm_f64
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import to_np64

pytestmark = pytest.mark.gpu


def _case(E, N, K, g, m, seed):
    ds = [synth.awq_like(1, N, K, group=g, seed=seed + e) for e in range(E)]
    qs = [d["q"] for d in ds]
    s = np.stack([d["s"] for d in ds])
    z = np.stack([d["z"] for d in ds])
    A = synth.awq_like(max(sum(m), 1), N, K, seed=seed + 99)["A"][:sum(m)]
    tq = [torch.from_numpy(q).cuda() for q in qs]
    ts, tz = torch.from_numpy(s).cuda(), torch.from_numpy(z).cuda()
    pe = api.pack_experts(tq, ts, tz, g)
    tA = torch.from_numpy(np.ascontiguousarray(A, dtype=np.float32)).to(torch.bfloat16).cuda()
    C = api.gemm_w4a16_grouped(tA, pe, ts, tz, m)
    torch.cuda.synchronize()
    ref = grouped_gemm_f64(A, qs, s, z, g, m)
    # per-element bound with the largest dequantised weight over all experts
    r = compare.check(to_np64(C), ref, A, np.concatenate(qs, 0), np.concatenate(list(s), 0),
                      np.concatenate(list(z), 0), g, "bf16")
    return r, C


@pytest.mark.parametrize("m", [[5, 0, 3, 8, 1, 0, 11, 4], [16, 16, 0, 0, 0, 0, 16, 16], [1, 1, 1, 1, 1, 1, 1, 1]])
def test_mixtral_experts_grouped(m):
    """Mixtral-8x7B expert w1/w3 shape (CFG#4: N = 14336, K = 4096), 8 experts, decode routing."""
    r, _ = _case(8, 14336, 4096, 128, m, seed=4000)
    assert r["ok"], (m, compare.summary(r))


@pytest.mark.parametrize("g", [64, 128])
def test_many_experts_ragged_tokens(g):
    """64 experts, token counts 0..40 (token tiles of 64: two m-tile sizes, empty experts)."""
    rng = np.random.default_rng(7)
    m = [int(x) for x in rng.integers(0, 41, 64)]
    m[3] = 0
    r, _ = _case(64, 256, 512, g, m, seed=4100)
    assert r["ok"], compare.summary(r)


def test_deterministic_and_no_tokens_noop():
    m = [3, 0, 9, 2]
    r1, C1 = _case(4, 1024, 2048, 128, m, seed=4200)
    r2, C2 = _case(4, 1024, 2048, 128, m, seed=4200)
    assert r1["ok"] and torch.equal(C1, C2)
    pe = api.pack_experts([torch.zeros(256, 128, dtype=torch.uint8, device="cuda")] * 2,
                          torch.ones(2, 2, 128, dtype=torch.float16, device="cuda"),
                          torch.zeros(2, 2, 128, dtype=torch.float16, device="cuda"), 128)
    out = torch.empty(0, 128, dtype=torch.bfloat16, device="cuda")
    api.gemm_w4a16_grouped(torch.empty(0, 256, dtype=torch.bfloat16, device="cuda"), pe,
                           torch.ones(2, 2, 128, dtype=torch.float16, device="cuda"),
                           torch.zeros(2, 2, 128, dtype=torch.float16, device="cuda"), [0, 0], out=out)
