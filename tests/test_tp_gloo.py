"""Tensor-parallel host path, world size 2 over gloo on CPU (§8(e), reading R13).

Each rank shards the same seeded layer with tp.shard_bounds / tp.pad_k_to (the code the GPU
path uses), computes its shard's product with the ORACLE standing in for the kernel (the
library needs a B200), and exchanges results with the real torch.distributed collectives:

* column-parallel (N-shard): all_gather of the rank outputs == the unsharded oracle GEMM;
* row-parallel (K-shard): fp32 partials (the kernel's tm_gemm_w4a16_partial_f32 output type)
  summed by all_reduce, then one bf16 rounding (tm_tp_finalize) -> within the R12 bound of the
  unsharded oracle, and equal to rounding the fp32 sum computed locally in the same order;
* shard bounds tile [0, extent) exactly once across ranks, aligned to 128 columns / g rows.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import compare, gemm, numerics
from paper_2508_15601_b200 import synth, tp

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, M, N, K, group, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        d = synth.awq_like(M, N, K, group=group, seed=4242)  # same draw on every rank
        A, q, s, z = d["A"], d["q"], d["s"], d["z"]
        res = {}

        # shard bounds tile the extent exactly once
        nlo, nhi = tp.shard_bounds(N, WORLD, rank, 128)
        klo, khi = tp.shard_bounds(K, WORLD, rank, group)
        b = torch.tensor([nlo, nhi, klo, khi], dtype=torch.int64)
        allb = [torch.zeros_like(b) for _ in range(WORLD)]
        dist.all_gather(allb, b)
        res["bounds"] = torch.stack(allb).numpy()

        # column parallel: this rank's N-shard through the oracle, gathered
        c_loc = gemm.gemm_f64(A, q[:, nlo:nhi], s[:, nlo:nhi], z[:, nlo:nhi], group)
        parts = [torch.zeros(M, N // WORLD, dtype=torch.float64) for _ in range(WORLD)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(c_loc)))
        res["col"] = torch.cat(parts, dim=1).numpy()

        # row parallel: fp32 partial of this rank's K-shard, fp32 all-reduce, one bf16 rounding
        g0, g1 = klo // group, khi // group
        p64 = gemm.gemm_f64(A[:, klo:khi], q[klo:khi], s[g0:g1], z[g0:g1], group)
        part = torch.from_numpy(p64.astype(np.float32))
        mine = part.clone()
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        res["row_sum"] = part.numpy()
        res["row_bf16"] = numerics.round_bf16(part.numpy().astype(np.float64))
        allp = [torch.zeros_like(mine) for _ in range(WORLD)]
        dist.all_gather(allp, mine)
        res["row_parts"] = torch.stack(allp).numpy()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,N,K,group", [(3, 512, 1024, 128), (16, 768, 1536, 64)])
def test_tp_world2_gloo(tmp_path, M, N, K, group):
    port = _free_port()
    mp.start_processes(_worker, args=(port, M, N, K, group, str(tmp_path)), nprocs=WORLD, start_method="spawn",
                       join=True)
    r = [dict(np.load(tmp_path / f"rank{i}.npz")) for i in range(WORLD)]
    d = synth.awq_like(M, N, K, group=group, seed=4242)
    full = gemm.gemm_f64(d["A"], d["q"], d["s"], d["z"], group)

    # bounds: contiguous, aligned, covering
    bnd = r[0]["bounds"]
    assert bnd[0, 0] == 0 and bnd[-1, 1] == N and bnd[0, 2] == 0 and bnd[-1, 3] == K
    assert all(bnd[i, 1] == bnd[i + 1, 0] and bnd[i, 3] == bnd[i + 1, 2] for i in range(WORLD - 1))
    assert np.all(bnd[:, :2] % 128 == 0) and np.all(bnd[:, 2:] % group == 0)

    for i in range(WORLD):
        # column parallel reproduces the unsharded product (column slices of one definition)
        np.testing.assert_allclose(r[i]["col"], full, rtol=1e-12, atol=1e-12)
        # row parallel: every rank holds the same reduced sum, equal to the rank-order fp32 sum
        np.testing.assert_array_equal(r[i]["row_sum"], r[0]["row_sum"])
        parts = r[i]["row_parts"]
        np.testing.assert_array_equal(r[i]["row_sum"], parts[0] + parts[1])
        chk = compare.check(r[i]["row_bf16"], full, d["A"], d["q"], d["s"], d["z"], group, "bf16")
        assert chk["ok"], chk


def test_pad_k_to():
    assert tp.pad_k_to(4096, 2, 128) == 4096
    assert tp.pad_k_to(4000, 2, 128) == 4096
    assert tp.pad_k_to(14336, 8, 128) == 14336
    assert tp.pad_k_to(1, 4, 64) == 256
    with pytest.raises(ValueError):
        tp.shard_bounds(1000, 2, 0, 128)
