"""Tensor parallelism for the W4A16 GEMM (§8(e); "tensor parallelism", App. I).

Column-parallel (N-shard): rank r owns output columns [r*N/P, (r+1)*N/P) -- its slice of q,
s, z is packed on its own GPU; activations are replicated; no communication.
Row-parallel (K-shard): rank r owns reduction rows [r*K/P, (r+1)*K/P) (whole quantisation
groups) and the matching activation columns; it produces an fp32 partial with
tm_gemm_w4a16_partial_f32, the partials are summed with an fp32 all-reduce (NCCL over
NVLink on the GPU box, reading R13), and tm_tp_finalize rounds once to bf16.

The shard arithmetic here is plain index math (host side); the GEMM/finalize run in the
library.  `shard_bounds` is also what the CPU gloo tests check against the oracle.
"""

import torch
import torch.distributed as dist


def shard_bounds(extent, world, rank, align):
    """[lo, hi) of rank's contiguous shard of `extent`, every boundary a multiple of `align`.
    Raises if extent is not divisible into aligned shards (callers pad K with zero-weight
    groups first, reading R9)."""
    if extent % (world * align):
        raise ValueError(f"extent {extent} not divisible into {world} shards aligned to {align}")
    step = extent // world
    return rank * step, (rank + 1) * step


def pad_k_to(K, world, group):
    """Smallest K' >= K with K' % (world * group) == 0 (zero-weight groups pad the tail)."""
    unit = world * group
    return ((K + unit - 1) // unit) * unit


class ColumnParallelW4:
    """N-sharded W4A16 layer on this rank's GPU."""

    def __init__(self, q, s, z, group, world, rank):
        from . import api
        K, N = q.shape
        self.lo, self.hi = shard_bounds(N, world, rank, 128)
        self.s = s[:, self.lo:self.hi].contiguous()
        self.z = z[:, self.lo:self.hi].contiguous()
        self.packed = api.pack_w4(q[:, self.lo:self.hi].contiguous(), self.s, self.z, group)
        self.K, self.N = K, N

    def __call__(self, A, out=None):
        from . import api
        return api.gemm_w4a16(A, self.packed, self.s, self.z, out=out)


class RowParallelW4:
    """K-sharded W4A16 layer: fp32 partial + all-reduce + finalize."""

    def __init__(self, q, s, z, group, world, rank, process_group=None):
        from . import api
        K, N = q.shape
        self.lo, self.hi = shard_bounds(K, world, rank, group)
        g0, g1 = self.lo // group, self.hi // group
        self.s = s[g0:g1].contiguous()
        self.z = z[g0:g1].contiguous()
        self.packed = api.pack_w4(q[self.lo:self.hi].contiguous(), self.s, self.z, group)
        self.K, self.N = K, N
        self.pg = process_group

    def local_partial(self, A_shard, out=None):
        from . import api
        return api.gemm_w4a16_partial_f32(A_shard, self.packed, self.s, self.z, out=out)

    def __call__(self, A, partial=None, out=None):
        """A: full activations [M][K] (replicated); returns bf16 C [M][N] on every rank."""
        from . import api
        part = self.local_partial(A[:, self.lo:self.hi].contiguous() if A.shape[1] == self.K else A, out=partial)
        if dist.is_initialized() and dist.get_world_size(self.pg) > 1:
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.pg)
        return api.tp_finalize(part, out=out)


def allreduce_sum_fp32(t, group=None):
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def device_for_rank(local_rank):
    torch.cuda.set_device(local_rank)
    return torch.device("cuda", local_rank)
