"""Tensor parallelism for the W4A16 GEMM (§8(e); "tensor parallelism", App. I).

Column-parallel (N-shard): rank r owns output columns [r*N/P, (r+1)*N/P) -- its slice of q,
s, z is packed on its own GPU; activations are replicated; no communication.
Row-parallel (K-shard): rank r owns reduction rows [r*K/P, (r+1)*K/P) (whole quantisation
groups) and the matching activation columns; it produces an fp32 partial with
tm_gemm_w4a16_partial_f32, the partials are summed with an fp32 all-reduce (NCCL over
NVLink on the GPU box, reading R13), and tm_tp_finalize rounds once to bf16.

The shard arithmetic here is plain index math (host side); the GEMM/finalize run in the
library.  `shard_bounds` is also what the CPU gloo tests check against the oracle.

SymmReducer (§8(f) NEXT-1) replaces the all-reduce + finalize pair with the library's fused
kernel over torch symmetric memory: each rank's GEMM writes its fp32 partial straight into a
symmetric buffer, tm_tp_allreduce_finalize adds the ranks' partials (NVLS multimem.ld_reduce
through the multicast address when the fabric provides one, else a rank-ordered sum over the
peers' NVLink mappings) and rounds once to bf16 -- one launch of ours instead of NCCL + one.
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


class SymmReducer:
    """Fused TP all-reduce + finalize over a torch symmetric-memory fp32 buffer of max_elems."""

    def __init__(self, max_elems, group=None, device=None):
        import torch.distributed._symmetric_memory as symm_mem
        group = group or dist.group.WORLD
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.buf = symm_mem.empty(max_elems, dtype=torch.float32, device=device or torch.cuda.current_device())
        self.handle = symm_mem.rendezvous(self.buf, group.group_name)
        self.partial_ptrs = list(self.handle.buffer_ptrs)
        self.signal_ptrs = list(self.handle.signal_pad_ptrs)
        self.multicast_ptr = int(self.handle.multicast_ptr or 0)

    def partial(self, M, N):
        """This rank's fp32 partial [M][N] (the head of the symmetric buffer)."""
        return self.buf[:M * N].view(M, N)

    def finalize(self, M, N, out, stream=None):
        from . import api
        return api.tp_allreduce_finalize(self.partial_ptrs, self.signal_ptrs, self.multicast_ptr, self.rank,
                                         self.world, M * N, out, stream=stream)


class RowParallelW4:
    """K-sharded W4A16 layer: fp32 partial + all-reduce + finalize.  When K is not divisible into
    `world` shards of whole groups (Qwen2-72B down: K = 29568 = 231 groups of 128), K is padded to
    pad_k_to(K, world, group) with zero-weight groups (q = z = 0, s = 1; reading R9), so the
    padded columns of the activations contribute exactly 0."""

    def __init__(self, q, s, z, group, world, rank, process_group=None):
        from . import api
        K, N = q.shape
        Kp = pad_k_to(K, world, group)
        if Kp != K:
            q = torch.cat([q, q.new_zeros(Kp - K, N)])
            s = torch.cat([s, s.new_ones((Kp - K) // group, N)])
            z = torch.cat([z, z.new_zeros((Kp - K) // group, N)])
        self.lo, self.hi = shard_bounds(Kp, world, rank, group)
        g0, g1 = self.lo // group, self.hi // group
        self.s = s[g0:g1].contiguous()
        self.z = z[g0:g1].contiguous()
        self.packed = api.pack_w4(q[self.lo:self.hi].contiguous(), self.s, self.z, group)
        self.K, self.Kp, self.N = K, Kp, N
        self.pg = process_group

    def local_partial(self, A_shard, out=None):
        from . import api
        return api.gemm_w4a16_partial_f32(A_shard, self.packed, self.s, self.z, out=out)

    def shard_input(self, A):
        """This rank's columns of the full activations A [M][K] (zero-padded past K)."""
        if self.Kp != self.K:
            A = torch.nn.functional.pad(A, (0, self.Kp - self.K))
        return A[:, self.lo:self.hi].contiguous()

    def __call__(self, A, partial=None, out=None, reducer=None):
        """A: full activations [M][K] (replicated) or this rank's shard [M][hi - lo]; returns
        bf16 C [M][N] on every rank (reducer: a SymmReducer -> the fused NEXT-1 epilogue)."""
        from . import api
        A_loc = self.shard_input(A) if A.shape[1] == self.K else A
        if reducer is not None:
            M = A_loc.shape[0]
            if out is None:
                out = torch.empty(M, self.N, dtype=torch.bfloat16, device=A_loc.device)
            self.local_partial(A_loc, out=reducer.partial(M, self.N))
            return reducer.finalize(M, self.N, out)
        part = self.local_partial(A_loc, out=partial)
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
