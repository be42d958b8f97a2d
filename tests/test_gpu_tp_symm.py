"""GPU tests of the fused row-parallel epilogue (tm_tp_allreduce_finalize, §8(f) NEXT-1).

* pre-signalled peers, world P = 2..8 on one GPU: P partial buffers and signal pads in device
  memory, the peers' barrier words set before the launch (as if every peer had arrived), so
  one rank's kernel runs alone -- no kernels waiting on one another on one GPU.  The output
  must equal RNE_bf16 of the fp32 sum in rank order bit for bit (reading R13), including a
  count % 4 tail and count = 0; the kernel leaves its own pad words consumed (zero) and has
  raised its signal in every peer's pad;
* world = 1 through torch symmetric memory and the product classes (SymmReducer +
  RowParallelW4): bit-identical to tm_gemm_w4a16_partial_f32 + tm_tp_finalize and within the
  R12 bound of the fp64 oracle;
* the multicast (NVLS) path needs a multicast-capable fabric; on a box without one (one GPU:
  torch skips multicast) it is not exercised and the test says so.
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.gemm import gemm_f64
from oracle.numerics import round_to
from paper_2508_15601_b200 import api, synth, tp
from tests.gpu_helpers import bits16, to_dev, to_np64

pytestmark = pytest.mark.gpu

WORDS = 64  # TM_TP_SIGNAL_WORDS


def _presignalled(P, rank, count, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    parts = [torch.randn(max(count, 1), generator=g).float().cuda() * (r + 1) for r in range(P)]
    pads = [torch.zeros(WORDS * P, dtype=torch.int32, device="cuda") for _ in range(P)]
    for ch in range(WORDS):  # every peer t != rank has signalled this rank on every channel
        for t in range(P):
            if t != rank:
                pads[rank][ch * P + t] = 1
    out = torch.full((max(count, 1),), 7.0, dtype=torch.bfloat16, device="cuda")
    return parts, pads, out


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("count", [4096 * 16, 4096 * 16 + 3, 1])
def test_presignalled_rank_order_sum_bit_exact(P, count):
    rank = P - 1
    parts, pads, out = _presignalled(P, rank, count, seed=P * 100 + count)
    api.tp_allreduce_finalize([p.data_ptr() for p in parts], [s.data_ptr() for s in pads], 0, rank, P, count, out)
    torch.cuda.synchronize()
    acc = parts[0][:count].cpu().numpy().astype(np.float32)
    for r in range(1, P):
        acc = (acc + parts[r][:count].cpu().numpy().astype(np.float32)).astype(np.float32)
    want = round_to(acc.astype(np.float64), "bf16")
    assert np.array_equal(to_np64(out[:count]), want)
    own = pads[rank].cpu().numpy().reshape(WORDS, P)
    assert not own.any(), "the kernel must consume every signal addressed to it"
    for t in range(P):
        if t != rank:
            assert (pads[t].cpu().numpy().reshape(WORDS, P)[:, rank] == 1).all(), "signal raised in every peer pad"


def test_presignalled_count_zero_runs_barriers():
    P, rank = 2, 0
    parts, pads, out = _presignalled(P, rank, 0, seed=5)
    api.tp_allreduce_finalize([p.data_ptr() for p in parts], [s.data_ptr() for s in pads], 0, rank, P, 0, out)
    torch.cuda.synchronize()
    assert not pads[rank].cpu().numpy().any()
    assert float(out[0]) == 7.0  # nothing written


def test_invalid_arguments():
    t = torch.zeros(64, device="cuda")
    s = torch.zeros(64, dtype=torch.int32, device="cuda")
    o = torch.zeros(64, dtype=torch.bfloat16, device="cuda")
    for rank, world in ((0, 0), (1, 1), (0, 9)):
        with pytest.raises(api.TMError):
            api.tp_allreduce_finalize([t.data_ptr()] * max(world, 1), [s.data_ptr()] * max(world, 1), 0, rank, world, 64, o)
    with pytest.raises(api.TMError):  # misaligned partial
        api.tp_allreduce_finalize([t.data_ptr() + 4], [s.data_ptr()], 0, 0, 1, 32, o)


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.fixture
def world1_group():
    import torch.distributed as dist
    created = False
    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", torch.cuda.current_device()))
        created = True
    yield dist.group.WORLD
    if created:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,N,K", [(16, 4096, 4096), (1, 4096, 14336), (5, 1024, 2048)])
def test_world1_symm_reducer_row_parallel(world1_group, M, N, K):
    d = synth.awq_like(M, N, K, group=128, seed=4000 + M)
    t = to_dev(d)
    row = tp.RowParallelW4(t["q"], t["s"], t["z"], 128, 1, 0)
    red = tp.SymmReducer(16 * 8192, group=world1_group)
    C = row(t["A"], reducer=red)
    P = row.local_partial(t["A"])
    C_ref = api.tp_finalize(P)
    torch.cuda.synchronize()
    assert np.array_equal(bits16(C), bits16(C_ref))
    r = compare.check(to_np64(C), gemm_f64(d["A"], d["q"], d["s"], d["z"], 128), d["A"], d["q"], d["s"], d["z"],
                      128, "bf16")
    assert r["ok"], compare.summary(r)
    # back-to-back layers through the same reducer (pad words reused across calls)
    for _ in range(3):
        C2 = row(t["A"], reducer=red)
    torch.cuda.synchronize()
    assert np.array_equal(bits16(C2), bits16(C_ref))
    if red.multicast_ptr == 0:
        print("multicast (NVLS) not available on this box: rank-ordered peer sum exercised")
