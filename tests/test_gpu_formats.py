"""GPU: checkpoint converters (AWQ / GPTQ -> LAYOUT v1) bit-exact to the oracle, and the W8A16
GEMM (bit planes) against the plain 8-bit definition (§8(f) NEXT-4)."""

import numpy as np
import pytest
import torch

from oracle import compare, formats as F, layout_v1
from oracle.gemm import gemm_f64
from paper_2508_15601_b200 import api, synth
from tests.gpu_helpers import bits16, to_np64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,N,g", [(256, 384, 128), (4096, 4096, 128), (1024, 512, 64)])
def test_awq_converter_bit_exact(K, N, g):
    d = synth.uniform(1, N, K, group=g, seed=5000 + K)
    qw = F.awq_pack_cols(d["q"])
    qz = F.awq_pack_cols(d["z"].astype(np.uint8))
    p, z = api.pack_awq(torch.from_numpy(qw).cuda(), torch.from_numpy(qz).cuda(), K, N, g)
    torch.cuda.synchronize()
    q_ref, z_ref = F.awq_unpack(qw, qz, N)
    assert np.array_equal(p.data.cpu().numpy(), layout_v1.pack(q_ref))
    assert np.array_equal(bits16(z), z_ref.view(np.uint16))


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("K,N,g", [(256, 384, 128), (4096, 6144, 128), (1024, 512, 64)])
def test_gptq_converter_bit_exact(K, N, g, offset):
    d = synth.uniform(1, N, K, group=g, seed=5100 + K + offset)
    zz = np.clip(d["z"].astype(np.int64), offset, 15)
    qw, qz = F.gptq_pack(d["q"], zz, zero_offset=offset)
    p, z = api.pack_gptq(torch.from_numpy(qw).cuda(), torch.from_numpy(qz).cuda(), K, N, g, zero_offset=offset)
    torch.cuda.synchronize()
    q_ref, z_ref = F.gptq_unpack(qw, qz, N, zero_offset=offset)
    assert np.array_equal(p.data.cpu().numpy(), layout_v1.pack(q_ref))
    assert np.array_equal(bits16(z), z_ref.view(np.uint16))


def test_awq_checkpoint_gemm_end_to_end():
    """An AWQ-format layer through the converter and the GEMM vs the oracle on the decoded weight."""
    M, N, K, g = 16, 4096, 4096, 128
    d = synth.awq_like(M, N, K, group=g, seed=5200)
    qw, qz = F.awq_pack_cols(d["q"]), F.awq_pack_cols(d["z"].astype(np.uint8))
    p, z = api.pack_awq(torch.from_numpy(qw).cuda(), torch.from_numpy(qz).cuda(), K, N, g)
    s = torch.from_numpy(d["s"]).cuda()
    A = torch.from_numpy(np.ascontiguousarray(d["A"], dtype=np.float32)).to(torch.bfloat16).cuda()
    C = api.gemm_w4a16(A, p, s, z)
    torch.cuda.synchronize()
    r = compare.check(to_np64(C), gemm_f64(d["A"], d["q"], d["s"], d["z"], g), d["A"], d["q"], d["s"], d["z"], g,
                      "bf16")
    assert r["ok"], compare.summary(r)


def _w8_case(M, N, K, g, seed):
    rng = np.random.default_rng(seed)
    W = rng.normal(0, 0.02, (K // g, g, N)).astype(np.float32)
    mn, mx = W.min(axis=1), W.max(axis=1)
    s = np.maximum((mx - mn) / 255.0, 2.0 ** -14).astype(np.float16)
    z8 = np.clip(np.rint(-mn / s.astype(np.float32)), 0, 255).astype(np.int64)
    q8 = np.clip(np.rint(W / s.astype(np.float32)[:, None, :]) + z8[:, None, :], 0, 255).astype(np.uint8).reshape(K, N)
    A = rng.normal(size=(M, K)).astype(np.float32)
    A = torch.from_numpy(A).to(torch.bfloat16).float().numpy().astype(np.float64)
    return A, q8, s, z8


@pytest.mark.parametrize("M", [1, 16, 256])
@pytest.mark.parametrize("N,K,g", [(4096, 4096, 128), (6144, 4096, 64), (1024, 14336, 128)])
def test_w8a16_gemm(M, N, K, g):
    A, q8, s, z8 = _w8_case(M, N, K, g, 5300 + M + N)
    p, s4, z4 = api.pack_w8(torch.from_numpy(q8).cuda(), torch.from_numpy(s).cuda(),
                            torch.from_numpy(z8.astype(np.float16)).cuda(), g)
    tA = torch.from_numpy(A.astype(np.float32)).to(torch.bfloat16).cuda()
    C = api.gemm_w8a16(tA, p, s4, z4)
    torch.cuda.synchronize()
    # the planes the packer wrote are the oracle's bit planes (bit-exact), and the product meets R12
    q4, s4r, z4r = F.w8_bitplanes(q8, s, z8)
    assert np.array_equal(p.data.cpu().numpy(), layout_v1.pack(q4))
    assert np.array_equal(bits16(s4), s4r.view(np.uint16)) and np.array_equal(bits16(z4), z4r.view(np.uint16))
    ref = F.w8a16_gemm_f64(A, q8, s, z8, g)
    r = compare.check(to_np64(C), ref, np.concatenate([A, A], axis=1), q4, s4r, z4r, g, "bf16")
    assert r["ok"], compare.summary(r)
