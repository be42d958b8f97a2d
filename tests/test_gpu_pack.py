"""GPU parity: tm_pack_w4 / tm_unpack_w4 / tm_dequant_w4 bit-exact against the oracle."""

import numpy as np
import pytest
import torch

from oracle import layout_v1 as L
from oracle.quant import dequant_rounded
from oracle.numerics import bf16_bits, fp16_bits
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import bits16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,N,group", [(256, 256, 128), (64, 128, 64), (192, 384, 64), (1024, 640, 128)])
def test_pack_bit_exact(K, N, group):
    rng = np.random.default_rng(K + N)
    q = rng.integers(0, 256, size=(K, N), dtype=np.uint8)  # high nibble must be ignored
    s = np.ones((K // group, N), dtype=np.float16)
    z = np.zeros((K // group, N), dtype=np.float16)
    p = api.pack_w4(torch.from_numpy(q).cuda(), torch.from_numpy(s).cuda(), torch.from_numpy(z).cuda(), group)
    got = p.data.cpu().numpy()
    assert np.array_equal(got, L.pack(q))
    assert (p.desc.K, p.desc.N, p.desc.group, p.desc.layout) == (K, N, group, api.TM_LAYOUT_V1)
    assert np.array_equal(api.unpack_w4(p).cpu().numpy(), q & 0xF)


@pytest.mark.parametrize("K,N", [(4096, 28672), (14336, 4096), (8192, 10240)])
def test_pack_full_size_sampled_tiles(K, N):
    """Llama-3 shapes: GPU pack of the whole matrix; the oracle packs sampled n-tiles (an
    n-tile's blobs are contiguous in LAYOUT v1, so its bytes are a slice of the whole)."""
    g = torch.Generator(device="cuda").manual_seed(K ^ N)
    qd = torch.randint(0, 16, (K, N), dtype=torch.uint8, device="cuda", generator=g)
    s = torch.ones((K // 128, N), dtype=torch.float16, device="cuda")
    p = api.pack_w4(qd, s, s, 128)
    KS = K // 64
    tiles = sorted({0, N // 128 - 1, 1, (N // 128) // 2})
    for nt in tiles:
        qt = qd[:, nt * 128:(nt + 1) * 128].cpu().numpy()
        got = p.data[nt * KS * 4096:(nt + 1) * KS * 4096].cpu().numpy()
        assert np.array_equal(got, L.pack(qt)), nt
    # unpack is the exact inverse over the whole matrix
    assert torch.equal(api.unpack_w4(p), qd)


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
def test_dequant_exhaustive_bit_exact(dtype):
    """All 16 codes x 16 integer zeros x all 63,488 finite fp16 scales (+ and -), through
    tm_dequant_w4 (the GEMM's dequant code) vs oracle.quant.dequant_rounded (reading R6)."""
    pos = np.arange(0, 0x7C00, dtype=np.uint16)
    sbits = np.concatenate([pos, pos | 0x8000])          # 63,488 finite patterns
    N = sbits.size                                        # = 496 * 128
    group = 64
    K = 16 * group                                        # group g has zero point g
    q = np.tile((np.arange(K) % 16).astype(np.uint8)[:, None], (1, N))
    z = np.tile(np.arange(16, dtype=np.float16)[:, None], (1, N))
    s = np.tile(sbits.view(np.float16)[None, :], (16, 1))
    dq, ds, dz = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (q, s, z))
    p = api.pack_w4(dq, ds, dz, group)
    W = api.dequant_w4(p, ds, dz, dtype)
    got = bits16(W)
    for k0 in range(0, K, 128):  # chunk the oracle to bound memory
        ref = dequant_rounded(q[k0:k0 + 128], s[k0 // group:(k0 + 128) // group], z[k0 // group:(k0 + 128) // group],
                              group, dtype)
        ref_bits = bf16_bits(ref) if dtype == "bf16" else fp16_bits(ref)
        mism = np.nonzero(got[k0:k0 + 128] != ref_bits)
        assert mism[0].size == 0, (dtype, k0 + mism[0][:5], mism[1][:5])


def test_dequant_awq_like_matches_exact_closed_form():
    d = synth.awq_like(1, 256, 512, group=128, seed=5)
    dq, ds, dz = (torch.from_numpy(d[k]).cuda() for k in ("q", "s", "z"))
    p = api.pack_w4(dq, ds, dz, 128)
    for dt in ("bf16", "fp16"):
        got = api.dequant_w4(p, ds, dz, dt).float().cpu().numpy()
        assert np.array_equal(got.astype(np.float64), dequant_rounded(d["q"], d["s"], d["z"], 128, dt))


def test_error_codes():
    s = torch.ones((1, 128), dtype=torch.float16, device="cuda")
    with pytest.raises(api.TMError, match="UNSUPPORTED_SHAPE"):
        api.pack_w4(torch.zeros((100, 128), dtype=torch.uint8, device="cuda"), s, s, 64)
    with pytest.raises(api.TMError, match="UNSUPPORTED_SHAPE"):
        api.pack_w4(torch.zeros((128, 128), dtype=torch.uint8, device="cuda"), s, s, 32)
    assert api.pack_w4_bytes(4096, 4096, 128) == 4096 * 4096 // 2
