"""ctypes binding of libtm_w4a16.so (include/tm_w4a16.h, include/tm_w4a16_debug.h).
Argument marshalling only.

Every function here forwards torch CUDA tensors as raw device pointers plus the
current CUDA stream to the C ABI; all computation happens in the library's
kernels.  The library is loaded on first use; if it is missing or cannot be
loaded the call raises (there is no CPU or PyTorch fallback).
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# TM_LIB_PATH: an alternative build of the same library (A/B timing scripts); default in-tree
LIB_PATH = os.environ.get("TM_LIB_PATH") or os.path.join(_HERE, "libtm_w4a16.so")

TM_LAYOUT_V1 = 1
TM_LAYOUT_V1_W8 = 2
TM_DTYPE_BF16, TM_DTYPE_FP16, TM_DTYPE_F32 = 0, 1, 2
_DT = {torch.bfloat16: TM_DTYPE_BF16, torch.float16: TM_DTYPE_FP16, torch.float32: TM_DTYPE_F32}

_lib = None


class TMError(RuntimeError):
    pass


class tm_packed_w4(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("bytes", ctypes.c_int64),
        ("K", ctypes.c_int32),
        ("N", ctypes.c_int32),
        ("group", ctypes.c_int32),
        ("layout", ctypes.c_uint32),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_SIGS = {
    "tm_pack_w4_bytes": (ctypes.c_int64, [_I, _I, _I]),
    "tm_pack_w4": (_I, [_P, _P, _P, _I, _I, _I, ctypes.POINTER(tm_packed_w4), _P]),
    "tm_gemm_w4a16": (_I, [_P, ctypes.POINTER(tm_packed_w4), _P, _P, _P, _I, _I, _I, _P]),
    "tm_gemm_w4a16_f16": (_I, [_P, ctypes.POINTER(tm_packed_w4), _P, _P, _P, _I, _I, _I, _P]),
    "tm_gemm_w4a16_partial_f32": (_I, [_P, ctypes.POINTER(tm_packed_w4), _P, _P, _P, _I, _I, _I, _P]),
    "tm_gemm_workspace_bytes": (ctypes.c_int64, [_I, _I, _I, _I]),
    "tm_gemm_w4a16_ws": (_I, [_P, ctypes.POINTER(tm_packed_w4), _P, _P, _P, _I, _I, _I, _I, _I, _P,
                              ctypes.c_int64, _P]),
    "tm_debug_dequant_int": (_I, [ctypes.POINTER(tm_packed_w4), _P, _P, _I, _P]),
    "tm_pack_awq": (_I, [_P, _P, _I, _I, _I, ctypes.POINTER(tm_packed_w4), _P, _P]),
    "tm_pack_gptq": (_I, [_P, _P, _I, _I, _I, _I, ctypes.POINTER(tm_packed_w4), _P, _P]),
    "tm_pack_w8_bytes": (ctypes.c_int64, [_I, _I, _I]),
    "tm_pack_w8": (_I, [_P, _P, _P, _I, _I, _I, ctypes.POINTER(tm_packed_w4), _P, _P, _P]),
    "tm_gemm_w8a16": (_I, [_P, ctypes.POINTER(tm_packed_w4), _P, _P, _P, _I, _I, _I, _P]),
    "tm_attn_workspace_bytes": (ctypes.c_int64, [_I, _I, _I, _I]),
    "tm_attn_decode_kv8": (_I, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, ctypes.c_float, _I, _P, ctypes.c_int64,
                                _P]),
    "tm_gemm_w4a16_grouped": (_I, [_P, ctypes.POINTER(tm_packed_w4), _P, _P, _P, ctypes.POINTER(ctypes.c_int32), _I,
                                   _I, _I, _P]),
    "tm_tp_finalize": (_I, [_P, _P, ctypes.c_int64, _P]),
    "tm_tp_allreduce_finalize": (_I, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), _P, _I, _I,
                                      ctypes.c_int64, _P, _P]),
    "tm_unpack_w4": (_I, [ctypes.POINTER(tm_packed_w4), _P, _P]),
    "tm_dequant_w4": (_I, [ctypes.POINTER(tm_packed_w4), _P, _P, _P, _I, _P]),
    "tm_set_gemm_override": (_I, [_I, _I]),
    "tm_query_gemm_config": (_I, [_I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "tm_query_gemm_kind": (_I, [_I, _I, _I, ctypes.POINTER(_I)]),
    "tm_set_decode_cluster": (_I, [_I]),
    "tm_set_decode_path": (_I, [_I, _I]),
    "tm_set_prefill_persistent": (_I, [_I]),
    "tm_set_prefill_pair": (_I, [_I]),
    "tm_set_trace": (_I, [_P, ctypes.c_int64]),
    "tm_status_string": (ctypes.c_char_p, [_I]),
    "tm_version": (ctypes.c_char_p, []),
}


def lib():
    """Load (once) and return the ctypes handle; raises if the library is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TMError(f"{LIB_PATH} not built: run `python -m paper_2508_15601_b200.build` "
                          "(no fallback path exists)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            try:
                fn = getattr(handle, name)
            except AttributeError:
                if LIB_PATH.endswith(os.path.join("paper_2508_15601_b200", "libtm_w4a16.so")):
                    raise  # the in-tree build must export the whole header
                continue  # an older build under TM_LIB_PATH (A/B timing): calls to it fail later
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def _check(status):
    if status != 0:
        raise TMError(lib().tm_status_string(status).decode())


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
            raise TMError("expected contiguous CUDA tensors")


class PackedW4:
    """A packed weight: device buffer (torch uint8 tensor) + the C descriptor."""

    def __init__(self, data, K, N, group):
        self.data = data
        self.desc = tm_packed_w4(data.data_ptr(), data.numel(), 0, 0, 0, 0)
        self.K, self.N, self.group = K, N, group

    @property
    def nbytes(self):
        return self.data.numel()


def pack_w4_bytes(K, N, group):
    r = lib().tm_pack_w4_bytes(K, N, group)
    if r < 0:
        _check(int(r))
    return int(r)


def pack_w4(q, scales, zeros, group, stream=None, out=None):
    """tm_pack_w4: q uint8 [K][N], scales/zeros fp16 [K/group][N] -> PackedW4."""
    _require_cuda(q, scales, zeros)
    K, N = q.shape
    nbytes = pack_w4_bytes(K, N, group)
    data = out if out is not None else torch.empty(nbytes, dtype=torch.uint8, device=q.device)
    p = PackedW4(data, K, N, group)
    _check(lib().tm_pack_w4(_ptr(q), _ptr(scales), _ptr(zeros), K, N, group, ctypes.byref(p.desc), _stream(stream)))
    return p


def _gemm(fn, A, packed, scales, zeros, out, out_dtype, stream):
    _require_cuda(A, scales, zeros)
    M, K = A.shape
    N = packed.N
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=A.device)
    _require_cuda(out)
    _check(fn(_ptr(A), ctypes.byref(packed.desc), _ptr(scales), _ptr(zeros), _ptr(out), M, N, K, _stream(stream)))
    return out


def gemm_w4a16(A, packed, scales, zeros, out=None, stream=None):
    """tm_gemm_w4a16: bf16 A [M][K] x packed W -> bf16 C [M][N]."""
    return _gemm(lib().tm_gemm_w4a16, A, packed, scales, zeros, out, torch.bfloat16, stream)


def gemm_w4a16_f16(A, packed, scales, zeros, out=None, stream=None):
    """tm_gemm_w4a16_f16: fp16 A -> fp16 C."""
    return _gemm(lib().tm_gemm_w4a16_f16, A, packed, scales, zeros, out, torch.float16, stream)


def gemm_w4a16_partial_f32(A, packed, scales, zeros, out=None, stream=None):
    """tm_gemm_w4a16_partial_f32: bf16 A -> fp32 partial C (row-parallel TP)."""
    return _gemm(lib().tm_gemm_w4a16_partial_f32, A, packed, scales, zeros, out, torch.float32, stream)


def gemm_workspace_bytes(M, N, K, group):
    """tm_gemm_workspace_bytes: bytes of caller workspace tm_gemm_w4a16_ws needs (0: none)."""
    r = lib().tm_gemm_workspace_bytes(M, N, K, group)
    if r < 0:
        _check(int(r))
    return int(r)


def gemm_workspace(M, N, K, group, device="cuda"):
    """A zero-filled workspace tensor for tm_gemm_w4a16_ws (None when the shape needs none)."""
    n = gemm_workspace_bytes(M, N, K, group)
    return torch.zeros(n, dtype=torch.uint8, device=device) if n else None


def gemm_w4a16_ws(A, packed, scales, zeros, workspace, out=None, out_dtype=None, stream=None):
    """tm_gemm_w4a16_ws: explicit dtypes (A bf16/fp16; C = A's dtype or fp32) and a caller-owned
    workspace (torch uint8 CUDA tensor, zero-filled before first use, or None if not needed)."""
    _require_cuda(A, scales, zeros)
    M, K = A.shape
    out_dtype = out_dtype or A.dtype
    if out is None:
        out = torch.empty((M, packed.N), dtype=out_dtype, device=A.device)
    _require_cuda(out)
    wp, wb = (None, 0) if workspace is None else (_ptr(workspace), workspace.numel())
    _check(lib().tm_gemm_w4a16_ws(_ptr(A), ctypes.byref(packed.desc), _ptr(scales), _ptr(zeros), _ptr(out), M,
                                  packed.N, K, _DT[A.dtype], _DT[out.dtype], wp, wb, _stream(stream)))
    return out


def pack_awq(qweight, qzeros, K, N, group, stream=None):
    """tm_pack_awq: AWQ int4 checkpoint tensors -> (PackedW4, fp16 zeros [K/g][N])."""
    _require_cuda(qweight, qzeros)
    data = torch.empty(pack_w4_bytes(K, N, group), dtype=torch.uint8, device=qweight.device)
    z = torch.empty((K // group, N), dtype=torch.float16, device=qweight.device)
    p = PackedW4(data, K, N, group)
    _check(lib().tm_pack_awq(_ptr(qweight), _ptr(qzeros), K, N, group, ctypes.byref(p.desc), _ptr(z), _stream(stream)))
    return p, z


def pack_gptq(qweight, qzeros, K, N, group, zero_offset=1, stream=None):
    """tm_pack_gptq: GPTQ int4 checkpoint tensors -> (PackedW4, fp16 zeros [K/g][N])."""
    _require_cuda(qweight, qzeros)
    data = torch.empty(pack_w4_bytes(K, N, group), dtype=torch.uint8, device=qweight.device)
    z = torch.empty((K // group, N), dtype=torch.float16, device=qweight.device)
    p = PackedW4(data, K, N, group)
    _check(lib().tm_pack_gptq(_ptr(qweight), _ptr(qzeros), K, N, group, zero_offset, ctypes.byref(p.desc), _ptr(z),
                              _stream(stream)))
    return p, z


def pack_w8(q8, scales, zeros8, group, stream=None):
    """tm_pack_w8: uint8 codes [K][N] + fp16 s, z8 [K/g][N] -> (packed bit planes, s4, z4 [2K/g][N])."""
    _require_cuda(q8, scales, zeros8)
    K, N = q8.shape
    nb = lib().tm_pack_w8_bytes(K, N, group)
    if nb < 0:
        _check(int(nb))
    data = torch.empty(int(nb), dtype=torch.uint8, device=q8.device)
    s4 = torch.empty((2 * K // group, N), dtype=torch.float16, device=q8.device)
    z4 = torch.empty((2 * K // group, N), dtype=torch.float16, device=q8.device)
    p = PackedW4(data, 2 * K, N, group)
    _check(lib().tm_pack_w8(_ptr(q8), _ptr(scales), _ptr(zeros8), K, N, group, ctypes.byref(p.desc), _ptr(s4), _ptr(z4),
                            _stream(stream)))
    return p, s4, z4


def gemm_w8a16(A, packed8, s4, z4, out=None, stream=None):
    """tm_gemm_w8a16: bf16 A [M][K] x W8 (tm_pack_w8 outputs) -> bf16 C [M][N]."""
    _require_cuda(A, s4, z4)
    M, K = A.shape
    if out is None:
        out = torch.empty((M, packed8.N), dtype=torch.bfloat16, device=A.device)
    _require_cuda(out)
    _check(lib().tm_gemm_w8a16(_ptr(A), ctypes.byref(packed8.desc), _ptr(s4), _ptr(z4), _ptr(out), M, packed8.N, K,
                               _stream(stream)))
    return out


def attn_workspace(B, Hq, Hkv, Lmax, device="cuda"):
    """Zero-filled workspace tensor for tm_attn_decode_kv8 (None when not needed)."""
    n = lib().tm_attn_workspace_bytes(B, Hq, Hkv, Lmax)
    if n < 0:
        _check(int(n))
    return torch.zeros(int(n), dtype=torch.uint8, device=device) if n else None


def attn_decode_kv8(Q, k_codes, v_codes, k_sz, v_sz, seq_lens, workspace=None, scale=None, out=None, stream=None):
    """tm_attn_decode_kv8: Q [B][Hq][128] bf16/fp16, codes uint8 [B][Hkv][Lmax][128], sz uint32
    [B][Hkv][Lmax] (fp16 scale | zero << 16), seq_lens int32 [B] (device) -> O like Q."""
    _require_cuda(Q, k_codes, v_codes, k_sz, v_sz, seq_lens)
    B, Hq, D = Q.shape
    _, Hkv, Lmax, _ = k_codes.shape
    if out is None:
        out = torch.empty_like(Q)
    wp, wb = (None, 0) if workspace is None else (_ptr(workspace), workspace.numel())
    sc = float(scale if scale is not None else 1.0 / D ** 0.5)
    _check(lib().tm_attn_decode_kv8(_ptr(Q), _ptr(k_codes), _ptr(v_codes), _ptr(k_sz), _ptr(v_sz), _ptr(seq_lens),
                                    _ptr(out), B, Hq, Hkv, Lmax, sc, _DT[Q.dtype], wp, wb, _stream(stream)))
    return out


def pack_kv_sz(scale, zero):
    """fp16 scale and zero tensors [...] -> uint32 [...] (scale in the low half) for the KV cache."""
    s = scale.contiguous().view(torch.int16).to(torch.int32) & 0xFFFF
    z = zero.contiguous().view(torch.int16).to(torch.int32) & 0xFFFF
    return (s | (z << 16)).contiguous()


class PackedExperts:
    """E experts' LAYOUT v1 weights back to back in one device buffer + the grouped descriptor."""

    def __init__(self, data, E, K, N, group):
        self.data, self.E, self.K, self.N, self.group = data, E, K, N, group
        self.desc = tm_packed_w4(data.data_ptr(), data.numel(), K, N, group, TM_LAYOUT_V1)


def pack_experts(qs, scales, zeros, group, stream=None):
    """Pack expert e's codes qs[e] (uint8 [K][N]) into slice e of one buffer with tm_pack_w4.
    scales/zeros: fp16 [E][K/group][N] (contiguous)."""
    E = len(qs)
    K, N = qs[0].shape
    per = pack_w4_bytes(K, N, group)
    data = torch.empty(E * per, dtype=torch.uint8, device=qs[0].device)
    for e in range(E):
        pack_w4(qs[e], scales[e], zeros[e], group, stream=stream, out=data[e * per:(e + 1) * per])
    return PackedExperts(data, E, K, N, group)


def gemm_w4a16_grouped(A, packed_experts, scales, zeros, m_per_expert, out=None, stream=None):
    """tm_gemm_w4a16_grouped: A bf16 [sum m_e][K] grouped by expert -> C bf16 [sum m_e][N]."""
    _require_cuda(A, scales, zeros)
    pe = packed_experts
    counts = (ctypes.c_int32 * pe.E)(*[int(m) for m in m_per_expert])
    if out is None:
        out = torch.empty((A.shape[0], pe.N), dtype=torch.bfloat16, device=A.device)
    _require_cuda(out)
    _check(lib().tm_gemm_w4a16_grouped(_ptr(A), ctypes.byref(pe.desc), _ptr(scales), _ptr(zeros), _ptr(out), counts,
                                       pe.E, pe.N, pe.K, _stream(stream)))
    return out


def tp_finalize(x_f32, out=None, stream=None):
    """tm_tp_finalize: fp32 -> bf16 (RNE)."""
    _require_cuda(x_f32)
    if out is None:
        out = torch.empty(x_f32.shape, dtype=torch.bfloat16, device=x_f32.device)
    _check(lib().tm_tp_finalize(_ptr(x_f32), _ptr(out), x_f32.numel(), _stream(stream)))
    return out


def unpack_w4(packed, stream=None):
    out = torch.empty((packed.K, packed.N), dtype=torch.uint8, device=packed.data.device)
    _check(lib().tm_unpack_w4(ctypes.byref(packed.desc), _ptr(out), _stream(stream)))
    return out


def dequant_w4(packed, scales, zeros, dtype="bf16", stream=None):
    _require_cuda(scales, zeros)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    out = torch.empty((packed.K, packed.N), dtype=tdt, device=packed.data.device)
    _check(lib().tm_dequant_w4(ctypes.byref(packed.desc), _ptr(scales), _ptr(zeros), _ptr(out),
                               0 if dtype == "bf16" else 1, _stream(stream)))
    return out


def debug_dequant_int(packed, zeros, dtype="bf16", stream=None):
    """tm_debug_dequant_int: the decode kernel's MMA operand (q - z) for every weight."""
    _require_cuda(zeros)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    out = torch.empty((packed.K, packed.N), dtype=tdt, device=packed.data.device)
    _check(lib().tm_debug_dequant_int(ctypes.byref(packed.desc), _ptr(zeros), _ptr(out),
                                      0 if dtype == "bf16" else 1, _stream(stream)))
    return out


def tp_allreduce_finalize(partial_ptrs, signal_ptrs, multicast_ptr, rank, world, count, out, stream=None):
    """tm_tp_allreduce_finalize: out (bf16 CUDA tensor, >= count elements) = RNE(sum over ranks
    of the fp32 partials); pointers are this process's mappings of the symmetric buffers."""
    _require_cuda(out)
    P = (ctypes.c_void_p * len(partial_ptrs))(*[int(x) for x in partial_ptrs])
    S = (ctypes.c_void_p * len(signal_ptrs))(*[int(x) for x in signal_ptrs])
    if len(partial_ptrs) < world or len(signal_ptrs) < world:
        raise TMError("tp_allreduce_finalize: fewer pointers than ranks")
    _check(lib().tm_tp_allreduce_finalize(P, S, ctypes.c_void_p(int(multicast_ptr) or None), rank, world, int(count),
                                          _ptr(out), _stream(stream)))
    return out


def set_gemm_override(tile_m=0, split_k=0):
    _check(lib().tm_set_gemm_override(tile_m, split_k))


def query_gemm_config(M, N, K):
    t, s, g, k = _I(), _I(), _I(), _I()
    _check(lib().tm_query_gemm_config(M, N, K, ctypes.byref(t), ctypes.byref(s), ctypes.byref(g)))
    _check(lib().tm_query_gemm_kind(M, N, K, ctypes.byref(k)))
    return dict(tile_m=t.value, split_k=s.value, grid_ctas=g.value, kind=k.value)


def set_decode_cluster(cs=0):
    """Tests/benchmarks: 0 automatic, 1 never (stream-K), 2..8 forced CTAs per tile."""
    _check(lib().tm_set_decode_cluster(cs))


def set_decode_path(path=0, split=0):
    """Tests/benchmarks: decode kernel for M <= 16 -- 0 automatic (the TMEM kernel), 1 the TMEM
    decode kernel, 2 register-fed; split in 1..8 forces the register-fed kernel's cluster split,
    split < 0 its stream-K CTA count."""
    _check(lib().tm_set_decode_path(path, split))


def set_prefill_persistent(on=True):
    """Tests/benchmarks: run the persistent prefill kernel (kind 4) for M >= 1024."""
    _check(lib().tm_set_prefill_persistent(1 if on else 0))


def set_prefill_pair(on=True):
    """Tests/benchmarks: CTA-pair prefill kernel (kind 5, the default where it applies) on/off;
    on=2 also runs 17 <= M <= 64 on 64-token pair tiles (experiment); on=3 keeps 256-token tiles at
    M <= 128 (A/B)."""
    _check(lib().tm_set_prefill_pair(int(on) if not isinstance(on, bool) else (1 if on else 0)))


def set_trace(buf=None):
    """Debug: enable (torch int32 CUDA tensor) or disable (None) the per-CTA GEMM timeline."""
    if buf is None:
        _check(lib().tm_set_trace(None, 0))
    else:
        _check(lib().tm_set_trace(_ptr(buf), buf.numel() * buf.element_size()))


def version():
    return lib().tm_version().decode()
