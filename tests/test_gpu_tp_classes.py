"""GPU tests of the product tensor-parallel classes (paper_2508_15601_b200/tp.py; §8(e)).

* world = 1: ColumnParallelW4 / RowParallelW4 on one GPU against the fp64 oracle;
* world = P ranks emulated in one process (every rank's shard built with the class, its local
  fp32 partial computed by the kernel, the partials summed in rank order as the fp32 all-reduce
  would, then tm_tp_finalize): column shards concatenate bit-exactly to the 1-GPU output (same
  launch configuration per shard), row shards meet the R12 bound -- including the zero-weight
  K padding of a K that does not split into whole groups (Qwen2-72B down analog);
* real NCCL at world = 2 (skipped with fewer than 2 GPUs; gpurun boxes have one).
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import compare
from oracle.gemm import gemm_f64
from paper_2508_15601_b200 import api, synth, tp
from tests.gpu_helpers import bits16, to_dev, to_np64

pytestmark = pytest.mark.gpu


def test_world1_column_and_row_classes():
    d = synth.awq_like(16, 1024, 2048, group=128, seed=3001)
    t = to_dev(d)
    col = tp.ColumnParallelW4(t["q"], t["s"], t["z"], 128, 1, 0)
    row = tp.RowParallelW4(t["q"], t["s"], t["z"], 128, 1, 0)
    C_col = col(t["A"])
    C_row = row(t["A"])
    torch.cuda.synchronize()
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    for C in (C_col, C_row):
        r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], 128, "bf16")
        assert r["ok"], compare.summary(r)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_column_parallel_shards_concatenate_bit_exact(P):
    M, N, K = 16, 128 * 8 * 4, 4096
    d = synth.awq_like(M, N, K, group=128, seed=3002 + P)
    t = to_dev(d)
    shards = [tp.ColumnParallelW4(t["q"], t["s"], t["z"], 128, P, r)(t["A"]) for r in range(P)]
    torch.cuda.synchronize()
    full = torch.cat(shards, dim=1)
    # the same per-shard configuration on the unsharded weight, column block by column block
    ref_bits = []
    for r in range(P):
        lo, hi = tp.shard_bounds(N, P, r, 128)
        p = api.pack_w4(t["q"][:, lo:hi].contiguous(), t["s"][:, lo:hi].contiguous(), t["z"][:, lo:hi].contiguous(), 128)
        ref_bits.append(bits16(api.gemm_w4a16(t["A"], p, t["s"][:, lo:hi].contiguous(), t["z"][:, lo:hi].contiguous())))
    assert np.array_equal(bits16(full), np.concatenate(ref_bits, axis=1))
    r = compare.check(to_np64(full), gemm_f64(d["A"], d["q"], d["s"], d["z"], 128), d["A"], d["q"], d["s"], d["z"],
                      128, "bf16")
    assert r["ok"], compare.summary(r)


@pytest.mark.parametrize("P,K", [(2, 4096), (4, 14336), (8, 28672), (2, 384), (8, 29568)])
def test_row_parallel_partials_rank_order_sum(P, K):
    """K = 384 at P = 2 and K = 29568 (Qwen2-72B down, 231 groups) at P = 8 need zero-weight
    padding to whole groups per rank (pad_k_to)."""
    M, N = 8, 1024
    d = synth.awq_like(M, N, K, group=128, seed=3010 + P + K)
    t = to_dev(d)
    acc = None
    for r in range(P):
        layer = tp.RowParallelW4(t["q"], t["s"], t["z"], 128, P, r)
        assert layer.Kp % (P * 128) == 0 and layer.Kp >= K
        part = layer.local_partial(layer.shard_input(t["A"]))
        acc = part.clone() if acc is None else acc + part   # rank order, fp32 (the all-reduce)
    C = api.tp_finalize(acc)
    torch.cuda.synchronize()
    ref = gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
    r = compare.check(to_np64(C), ref, d["A"], d["q"], d["s"], d["z"], 128, "bf16")
    assert r["ok"], (P, K, compare.summary(r))


def _nccl_worker(rank, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=2)
    d = synth.awq_like(8, 1024, 4096, group=128, seed=3050)
    t = to_dev(d)
    C = tp.RowParallelW4(t["q"], t["s"], t["z"], 128, 2, rank)(t["A"])
    torch.cuda.synchronize()
    if rank == 0:
        np.save(out, to_np64(C))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NCCL all-reduce over NVLink)")
def test_row_parallel_nccl_world2(tmp_path):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "c.npy")
    mp.spawn(_nccl_worker, args=(port, out), nprocs=2, join=True)
    d = synth.awq_like(8, 1024, 4096, group=128, seed=3050)
    r = compare.check(np.load(out), gemm_f64(d["A"], d["q"], d["s"], d["z"], 128), d["A"], d["q"], d["s"], d["z"],
                      128, "bf16")
    assert r["ok"], compare.summary(r)
