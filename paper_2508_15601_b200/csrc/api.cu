// api.cu -- host side of libtm_w4a16.so: the C ABI declared in include/tm_w4a16.h.
// Validation, launch-configuration choice, TMA descriptor encoding (cached), launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/tm_w4a16.h"
#include "../../include/tm_w4a16_debug.h"
#include "aux_kernels.cuh"
#include "gemm_w4a16.cuh"
#include "gemm_dec.cuh"
#include "gemm_rf.cuh"
#include "gemm_pk.cuh"
#include "gemm_2sm.cuh"
#include "attn_dec.cuh"
#include "tp_reduce.cuh"

namespace {

using namespace w4k;

constexpr int kNumSMsDefault = 148;

std::atomic<int> g_override_tile{0};
std::atomic<int> g_override_split{0};
std::atomic<int> g_dec_cluster{0};
std::atomic<int> g_dec_path{0};   // 0 automatic (the TMEM decode kernel), 1 TMEM decode kernel, 2 register-fed
std::atomic<int> g_rf_split{0};   // register-fed kernel: CTAs per tile (0 = automatic)
 // 0 automatic, 1 never (stream-K), 2..8 forced size,
                                     // -1 one CTA per tile (no split)
uint32_t* g_trace = nullptr;  // debug timeline buffer (tm_set_trace)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

tm_status check_shape(int K, int N, int group) {
  if (K <= 0 || N <= 0) return TM_ERR_INVALID_ARG;
  if (group != 64 && group != 128) return TM_ERR_UNSUPPORTED_SHAPE;
  if (N % 128 || K % 64 || K % group) return TM_ERR_UNSUPPORTED_SHAPE;
  return TM_OK;
}

tm_status from_cuda(cudaError_t e) { return e == cudaSuccess ? TM_OK : TM_ERR_CUDA; }

// Everything cached about a device (SM count, configured kernel attributes, occupancy, the
// library workspace) is kept per device ordinal: one process may drive several GPUs.
constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    (void)cudaGetLastError();
    return 0;
  }
  return dev;
}

int num_sms() {
  static std::atomic<int> sms[kMaxDevices] = {};
  const int dev = current_device();
  int v = sms[dev].load();
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
    (void)cudaGetLastError();
    return kNumSMsDefault;  // no device (host-side configuration queries): B200
  }
  sms[dev].store(v);
  return v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
template <typename Kern>
tm_status ensure_smem(Kern kern, int bytes, std::atomic<int> (&done)[kMaxDevices]) {
  const int dev = current_device();
  if (done[dev].load() >= bytes) return TM_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
    (void)cudaGetLastError();  // do not leave a stale error for the next launch check
    return TM_ERR_CUDA;
  }
  done[dev].store(bytes);
  return TM_OK;
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

struct MapKey {
  const void* ptr;
  int M, K, NT, bf16;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && M == o.M && K == o.K && NT == o.NT && bf16 == o.bf16;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.ptr);
    h ^= (static_cast<size_t>(k.M) * 0x9E3779B97F4A7C15ull) ^ (static_cast<size_t>(k.K) << 20) ^
         (static_cast<size_t>(k.NT) << 40) ^ static_cast<size_t>(k.bf16);
    return h;
  }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

tm_status act_tensor_map(const void* A, int M, int K, int NT, bool bf16, CUtensorMap* out) {
  const MapKey key{A, M, K, NT, bf16 ? 1 : 0};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return TM_OK;
    }
  }
  auto enc = get_encode();
  if (!enc) return TM_ERR_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(NT)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                   const_cast<void*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return TM_ERR_CUDA;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps.emplace(key, map);
  }
  *out = map;
  return TM_OK;
}

// 2-D output map for the tiled kernel's TMA-store epilogue: dims {N, M}, box {128, rows}
tm_status out_tensor_map(void* C, int M, int N, int NT, int esize, bool bf16, CUtensorMap* out) {
  const MapKey key{C, M, N, 1000 + NT * 8 + esize, bf16 ? 1 : 0};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return TM_OK;
    }
  }
  auto enc = get_encode();
  if (!enc) return TM_ERR_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(N) * esize};
  const int rows = esize == 4 && NT > 128 ? 128 : (NT < 256 ? NT : 256);
  const cuuint32_t box[2] = {128, static_cast<cuuint32_t>(rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                           : (bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  CUresult r = enc(&map, dt, 2, C, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return TM_ERR_CUDA;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps.emplace(key, map);
  }
  *out = map;
  return TM_OK;
}

// 3-D activation map for the stream-K kernel: dims {64, M, K/64}, strides {2K, 128} bytes,
// box {64, NT, CH/64}: one request lands CH/64 SW128 sub-tiles of NT x 64.
tm_status act_tensor_map_3d(const void* A, int M, int K, int NT, int blobs, bool bf16, CUtensorMap* out) {
  const MapKey key{A, M, K, NT | (blobs << 16) | (1 << 30), bf16 ? 1 : 0};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return TM_OK;
    }
  }
  auto enc = get_encode();
  if (!enc) return TM_ERR_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(K / 64)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 2, 128};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(NT), static_cast<cuuint32_t>(blobs)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                   const_cast<void*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return TM_ERR_CUDA;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps.emplace(key, map);
  }
  *out = map;
  return TM_OK;
}

// 2-D map over s or z ([K/g][N] fp16): box {128 columns, rows groups} (default 8).
tm_status sz_tensor_map(const void* p, int G, int N, CUtensorMap* out, int rows = 8) {
  const MapKey key{p, G, N, rows | (2 << 30), 2};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return TM_OK;
    }
  }
  auto enc = get_encode();
  if (!enc) return TM_ERR_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(G)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(N) * 2};
  const cuuint32_t box[2] = {128, static_cast<cuuint32_t>(rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(p), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return TM_ERR_CUDA;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps.emplace(key, map);
  }
  *out = map;
  return TM_OK;
}

// 2-D map over an 8-bit KV cache viewed as uint8 rows of 128 codes: box {128, 64 tokens}, SW128.
tm_status kv_tensor_map(const void* p, long long rows, CUtensorMap* out) {
  const MapKey key{p, static_cast<int>(rows & 0x7fffffff), static_cast<int>(rows >> 31), 64 | (3 << 28), 3};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return TM_OK;
    }
  }
  auto enc = get_encode();
  if (!enc) return TM_ERR_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, 64};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(p), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return TM_ERR_CUDA;
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps.emplace(key, map);
  }
  *out = map;
  return TM_OK;
}

// ---------------------------------------------------------------- stream-K workspace
// The stream-K decode kernel needs [flags: one int per CTA, 256-B aligned][fp32 partial slots:
// one NT x 128 tile per CTA].  Flags are zero between launches: the kernel returns every flag
// it raised to zero before it exits.  Callers either pass their own buffer (tm_gemm_w4a16_ws;
// zero-filled once before its first use) or use the library-owned one below.
size_t ws_flag_bytes(int ctas) { return (static_cast<size_t>(ctas) * sizeof(int) + 255) & ~size_t(255); }

// Library-owned workspace of the convenience entry points: one per (device, stream), allocated
// on first use (outside CUDA-graph capture) and grown when a larger shape class needs more.
struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
};
struct WsKey {
  int dev;
  cudaStream_t stream;
  int kind;  // 0: TMEM decode kernels (flags zero between launches), 1: register-fed kernel
             // (self-validating partial words, all zero between launches: never shared)
  bool operator==(const WsKey& o) const { return dev == o.dev && stream == o.stream && kind == o.kind; }
};
struct WsKeyHash {
  size_t operator()(const WsKey& k) const { return reinterpret_cast<size_t>(k.stream) * 31u + k.dev * 7u + k.kind; }
};
std::mutex g_ws_mu;
std::unordered_map<WsKey, Workspace, WsKeyHash> g_ws;

tm_status library_workspace(cudaStream_t stream, size_t need, void** out, int kind = 0) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  Workspace& w = g_ws[WsKey{current_device(), stream, kind}];
  if (w.bytes < need) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      (void)cudaGetLastError();
      return TM_ERR_CUDA;  // first use of a shape class must happen outside graph capture
    }
    if (w.ptr) {
      if (cudaStreamSynchronize(stream) != cudaSuccess) return TM_ERR_CUDA;
      cudaFree(w.ptr);
      w.ptr = nullptr;
      w.bytes = 0;
    }
    size_t alloc = need < (size_t(4) << 20) ? (size_t(4) << 20) : need;
    if (cudaMalloc(&w.ptr, alloc) != cudaSuccess) {
      (void)cudaGetLastError();
      return TM_ERR_CUDA;
    }
    // zeroed in stream order: a cudaMemset on the legacy stream does not order against non-blocking
    // streams, and the kernel reads the flags (measured: a stream-K launch on a fresh stream trapped)
    if (cudaMemsetAsync(w.ptr, 0, alloc, stream) != cudaSuccess) return TM_ERR_CUDA;
    w.bytes = alloc;
  }
  *out = w.ptr;
  return TM_OK;
}

// flags + partials for `ctas` CTAs of NT-token tiles, from the caller's buffer or the library's
tm_status get_workspace(cudaStream_t stream, void* user, int64_t user_bytes, int ctas, int nt, int** flags,
                        float** partials, int kind = 0) {
  const size_t fb = ws_flag_bytes(ctas);
  const size_t need = fb + static_cast<size_t>(ctas) * nt * 128 * sizeof(float);
  void* base = user;
  if (user) {
    if (user_bytes < static_cast<int64_t>(need)) return TM_ERR_INVALID_ARG;
    if (!aligned16(user)) return TM_ERR_MISALIGNED;
  } else {
    tm_status st = library_workspace(stream, need, &base, kind);
    if (st != TM_OK) return st;
  }
  *flags = static_cast<int*>(base);
  *partials = reinterpret_cast<float*>(static_cast<uint8_t*>(base) + fb);
  return TM_OK;
}

// ---------------------------------------------------------------- launch configuration
struct Config {
  int kind;  // 0 = classic tiles (+ cluster split-K), 1 = persistent stream-K, 4 = persistent
             // prefill (gemm_pk.cuh), 3 = register-fed
             // decode kernel (split = CTAs per tile), 2 = decode kernel
             // with CS CTAs per tile reduced over a thread-block cluster (split = CS)
  int NT;
  int split;  // classic: CTAs per tile along K; stream-K: number of persistent CTAs
  int grid_x, grid_y;
};

int sk_chunk(int nt) { return nt <= 64 ? 256 : (nt <= 128 ? 128 : 64); }

int max_split_for(int nt) {
  switch (nt) {
    case 16: return GemmCfg<16>::MAX_SPLIT;
    case 32: return GemmCfg<32>::MAX_SPLIT;
    case 64: return GemmCfg<64>::MAX_SPLIT;
    case 128: return GemmCfg<128>::MAX_SPLIT;
    default: return GemmCfg<256>::MAX_SPLIT;
  }
}

// how many clusters of `cs` decode CTAs can be resident at once (one wave); cached per (nt, cs)
template <int NT>
int dec_active_clusters_t(int cs) {
  static std::atomic<int> cache[kMaxDevices][9] = {};
  const int dev = current_device();
  int v = cache[dev][cs].load();
  if (v) return v;
  auto kern = w4a16_dec_kernel<NT, true, OUT_ACT>;
  const int fallback = num_sms() / cs;  // no device (host-side query): ideal packing
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DecCfg<NT>::SMEM) != cudaSuccess) {
    (void)cudaGetLastError();
    return fallback > 0 ? fallback : 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs * 64, 1, 1);
  cfg.blockDim = dim3(DecCfg<NT>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = DecCfg<NT>::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    n = fallback;
  }
  if (n < 1) n = 1;
  cache[dev][cs].store(n);
  return n;
}
int dec_active_clusters(int nt, int cs) {
  switch (nt) {
    case 16: return dec_active_clusters_t<16>(cs);
    case 32: return dec_active_clusters_t<32>(cs);
    case 64: return dec_active_clusters_t<64>(cs);
  }
  return 0;
}

int dec_max_cluster(int nt) {
  switch (nt) {
    case 16: return DecCfg<16>::MAX_CLUSTER;
    case 32: return DecCfg<32>::MAX_CLUSTER;
    case 64: return DecCfg<64>::MAX_CLUSTER;
  }
  return 1;
}

// fewest 256-k chunks a cluster-split CTA may own (experiments: TM_DEC_MIN_CHUNKS)
int dec_min_chunks() {
  static const int v = [] {
    const char* e = std::getenv("TM_DEC_MIN_CHUNKS");
    return e ? std::atoi(e) : 8;
  }();
  return v;
}

// Decode kernel launch shape for `tiles` output tiles of NT tokens x 128 columns over K.
// A few tiles (o/qkv/down-sized N) -> CS CTAs per tile in one cluster, reduced in distributed
// shared memory (no global flags, no gpu-scope fences); else persistent stream-K.  Measured on
// Llama-3-8B decode shapes: fixed per-CTA costs make ~8+ chunks of 256 k per CTA the sweet spot
// -- o_proj 64 CTAs 6.6 us vs 128 CTAs 7.0 us vs stream-K 8.1 us -- and a cluster layout that
// does not fit one wave is ~1.5x slower.
Config decode_config(int nt, int tiles, int K) {
  Config c{};
  c.NT = nt;
  const int kc = (K + 255) / 256;
  const int force = g_dec_cluster.load();
  const int cmax = dec_max_cluster(nt);
  int cs = 0;
  if (force >= 2) {
    cs = force < cmax ? force : cmax;
    if (cs > kc) cs = kc;
  } else if (force == -1) {
    cs = 1;
  } else if (force == 0) {
    for (int k = cmax; k >= 2; --k) {
      if (k > kc || (kc + k - 1) / k < dec_min_chunks() || tiles * k > num_sms()) continue;
      if (tiles > dec_active_clusters(nt, k)) continue;
      cs = k;
      break;
    }
  }
  if (cs == 0 && force == 0 && tiles <= num_sms() && tiles * 10 >= 7 * num_sms()) {
    // 70-100 % of the SMs have a whole tile each: one CTA per tile without a split beats
    // stream-K's fix-ups (measured Mixtral expert N=14336 K=4096, 112 tiles, M=16:
    // 12.5 -> 10.9 us at g=128; at 80 tiles -- Llama-3-70B qkv -- stream-K stays faster)
    cs = 1;
  }
  if (cs >= 1) {
    c.kind = 2;
    c.split = cs;
    c.grid_x = tiles * cs;
    c.grid_y = 1;
    return c;
  }
  // persistent stream-K: one CTA per SM, equal chunk ranges
  c.kind = 1;
  const long long total = static_cast<long long>(tiles) * kc;
  long long P = num_sms();
  if (P > total) P = total;
  c.split = static_cast<int>(P);
  c.grid_x = c.split;
  c.grid_y = 1;
  return c;
}

// clusters of `cs` register-fed CTAs that fit the GPU at once (cudaOccupancyMaxActiveClusters;
// per device, per cluster size; the NT = 16 / g = 64 instantiation has the largest footprint)
int rf_active_clusters(int cs) {
  static std::atomic<int> cache[kMaxDevices][9] = {};
  const int dev = current_device();
  if (cs < 1 || cs > 8) return 0;
  int v = cache[dev][cs].load();
  if (v > 0) return v;
  auto kern = w4a16_rf_kernel<16, 64, true, OUT_ACT>;
  static std::atomic<int> configured[kMaxDevices] = {};
  const bool smem_ok = ensure_smem(kern, RfCfg<16, 64>::SMEM, configured) == TM_OK;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs * 64, 1, 1);
  cfg.blockDim = dim3(RfCfg<16, 64>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = RfCfg<16, 64>::SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (!smem_ok || cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = (2 * num_sms()) / cs;  // (no device: the CPU-side query of the config)
  }
  cache[dev][cs].store(n);
  return n;
}

// Register-fed decode kernel (gemm_rf.cuh), M <= 16, in one wave at two CTAs per SM (the
// kernel's footprint allows two; under PDL the next launch's CTAs fill the SMs this launch leaves):
//  * few tiles (tiles <= SMs): S CTAs per tile in one cluster, DSMEM reduction -- the largest
//    S <= 8 with tiles x S <= 2 x SMs, >= 2 chunks of 256 k per CTA and all clusters resident;
//  * many tiles: stream-K over tiles x chunks with P = 2 x SMs CTAs (every SM equally loaded: the
//    register-fed inner loop runs at ~1.2x an SM's share of HBM, so imbalance costs directly),
//    partial tiles added in CTA order by the last contributor.
// Config: split = S (cluster) or -P (stream-K); debug override g_rf_split (> 0: S, < 0: -P).
Config rf_config(int M, int N, int K) {
  Config c{};
  c.kind = 3;
  c.NT = M <= 8 ? 8 : 16;
  const int tiles = N / 128;
  const int kc = (K + 255) / 256;
  const long long T = static_cast<long long>(tiles) * kc;
  int S = g_rf_split.load();
  if (S == 0) {
    if (tiles <= num_sms()) {
      S = 1;
      for (int s = 8; s >= 2; --s)
        if (tiles * s <= 2 * num_sms() && kc >= 2 * s && tiles <= rf_active_clusters(s)) {
          S = s;
          break;
        }
    } else {
      S = -2 * num_sms();
    }
  }
  if (S > 0) {
    if (S > 8) S = 8;
    if (S > kc) S = kc;
    c.split = S;
    c.grid_x = tiles * S;
  } else {
    long long P = -static_cast<long long>(S);
    if (P > T) P = T;
    c.split = -static_cast<int>(P);
    c.grid_x = static_cast<int>(P);
  }
  c.grid_y = 1;
  return c;
}

// The register-fed kernel is opt-in (tm_set_decode_path(2, ...)): measured on the CFG#1 decode
// shapes (scripts/rf_perf.py) it ties the TMEM kernel at M <= 8 on o/qkv and is
// slower on gate_up/down and at M = 16, so automatic dispatch keeps the TMEM kernel.
bool use_rf(int M) { return M <= 16 && g_dec_path.load() == 2; }



// Persistent prefill kernel (gemm_pk.cuh, kind 4): 128 x 192 tiles, one CTA per SM walking the
// tiles, double-buffered TMEM accumulator, for M >= kPkMinM (bf16/fp16 outputs; fp32 partials keep
// the tiled kernel).  Opt-in (tm_set_prefill_persistent): measured 7-30 % slower than the tiled
// kernel on every CFG#2 shape -- the stage loads, not the per-tile overheads, bound it.
constexpr int kPkNT = 192;
constexpr int kPkMinM = 1024;
std::atomic<int> g_pk{0};
bool use_pk(int M) {
  return g_pk.load() != 0 && M >= kPkMinM && g_override_tile.load() == 0 && g_override_split.load() == 0;
}
Config pk_config(int M, int N) {
  Config c{};
  c.kind = 4;
  c.NT = kPkNT;
  c.split = 1;
  const long long tiles = static_cast<long long>(N / 128) * ((M + kPkNT - 1) / kPkNT);
  c.grid_x = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
  c.grid_y = 1;
  return c;
}

// clusters of `cs` pair-kernel CTAs that fit the GPU at once (one CTA per SM; clusters of 6-8
// CTAs pack into the GPCs with leftovers, so fewer than SMs / cs -- a second wave of clusters
// doubled the mid-M split-K time when this was not checked)
template <int NT>
int pair_active_clusters(int cs) {
  static std::atomic<int> cache[kMaxDevices][9] = {};
  const int dev = current_device();
  if (cs < 2 || cs > 8) return 0;
  int v = cache[dev][cs].load();
  if (v > 0) return v;
  auto kern = w4a16_gemm_2sm_kernel<NT, true, OUT_ACT>;
  static std::atomic<int> configured[kMaxDevices] = {};
  const bool smem_ok = ensure_smem(kern, PairCfg<NT>::SMEM, configured) == TM_OK;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs * 32, 1, 1);
  cfg.blockDim = dim3(PairCfg<NT>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = PairCfg<NT>::SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (!smem_ok || cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = num_sms() / cs;  // (no device: the CPU-side query of the config)
  }
  cache[dev][cs].store(n);
  return n;
}

// CTA-pair prefill kernel (gemm_2sm.cuh, kind 5): where the tiled chooser picks 256-token tiles
// without split-K and N % 256 == 0 (bf16/fp16 outputs and fp32 partials).
// Measured 4-9 % faster than the tiled kernel on every CFG#2 shape; on by
// default, tm_set_prefill_pair(0) restores the tiled kernel (A/B, tests).
std::atomic<int> g_pair{1};
std::atomic<int> g_pair128{1};  // (A/B: tm_set_prefill_pair(3) = 256-token tiles for M <= 128 too)

Config choose_config_tiled(int M, int N, int K);
Config choose_config(int M, int N, int K) {
  if (use_rf(M)) return rf_config(M, N, K);
  if (use_pk(M)) return pk_config(M, N);
  Config c = choose_config_tiled(M, N, K);
  if (g_pair.load() == 0 || N % 256 != 0 || g_override_tile.load() != 0 || g_override_split.load() != 0) return c;
  if (c.kind == 0 && c.split == 1 && c.NT == Pair2Cfg::NT) {
    c.kind = 5;  // same grid: N / 128 CTAs (pairs along N) x M / 256
  } else if (c.kind == 0 && M > 64 && M <= 512) {
    // mid M: few pair tiles -> split K over up to 4 pairs of one cluster (2 S <= 8 CTAs,
    // reduced through distributed shared memory) while the clusters fit one wave; M <= 128 on
    // 128-token pair tiles (half the MMA work of a 256-token tile)
    const int ntile = (M <= 128 && g_pair128.load() != 0) ? 128 : 256;
    const int pairs = (N / 256) * ((M + ntile - 1) / ntile);
    const int KS = K / 64;
    int S = 1;
    for (int k = 4; k >= 2; --k) {
      const int act = ntile == 128 ? pair_active_clusters<128>(2 * k) : pair_active_clusters<256>(2 * k);
      if (pairs <= act && KS >= 4 * k) {
        S = k;
        break;
      }
    }
    if (S == 1) return c;  // no split fits: the tiled kernel's smaller tiles (gate_up M = 128: 45 vs 55 us)
    c.kind = 5;
    c.NT = ntile;
    c.split = S;
    c.grid_x = (N / 128) * S;
    c.grid_y = (M + ntile - 1) / ntile;
  } else if (g_pair.load() >= 2 && (c.kind == 1 || c.kind == 2) && M > 16 && M <= 64) {
    // small M on 64-token pair tiles (M = 256 x N = 64 MMAs), split K over up to 4 pairs
    const int pairs = N / 256;
    const int KS = K / 64;
    int S = 1;
    for (int k = 4; k >= 2; --k)
      if (pairs <= pair_active_clusters<64>(2 * k) && KS >= 4 * k) {
        S = k;
        break;
      }
    if (S == 1) return c;
    c.kind = 5;
    c.NT = 64;
    c.split = S;
    c.grid_x = (N / 128) * S;
    c.grid_y = 1;
  }
  return c;
}

Config choose_config_tiled(int M, int N, int K) {
  Config c{};
  int nt = 16;
  const int ot = g_override_tile.load();
  if (ot > 0) {
    nt = ot;
  } else if (M <= 16) {
    nt = 16;
  } else if (M <= 32) {
    nt = 32;
  } else if (M <= 64) {
    nt = 64;
  } else if (M <= 128 || (M <= 256 && 2 * (N / 128) <= num_sms())) {
    // (mid M: 128-token tiles while 2 m-tiles of them still fit one wave -- measured o_proj
    // M=256 23.7 us at NT=128 + split 2 vs 29.0 us at NT=256)
    nt = 128;
  } else {
    nt = 256;
  }
  const int n_tiles = N / 128;
  c.NT = nt;
  const int m_tiles = (M + nt - 1) / nt;
  const int KS = K / 64;
  int split = 1;
  const int os = g_override_split.load();
  if (os == 0 && nt <= 64) return decode_config(nt, n_tiles * m_tiles, K);
  if (os < 0 || (os == 0 && nt <= 64)) {
    // persistent stream-K: one CTA per SM (or -os CTAs when forced), equal chunk ranges
    c.kind = 1;
    const int ch = sk_chunk(nt);
    const long long total = static_cast<long long>(m_tiles) * n_tiles * ((K + ch - 1) / ch);
    long long P = os < 0 ? -os : num_sms();
    if (P > total) P = total;
    c.split = static_cast<int>(P);
    c.grid_x = c.split;
    c.grid_y = 1;
    return c;
  }
  c.kind = 0;
  if (os > 0) {
    split = os;
  } else if (nt <= 64) {
    // decode: fill ~2 CTAs per SM with split-K over a cluster (<= 8, portable)
    const int tiles = n_tiles * m_tiles;
    const int target = 2 * num_sms();
    split = (target + tiles - 1) / tiles;
    if (split > 8) split = 8;
  } else {
    // mid M: few tiles leave SMs idle while every CTA dequantises its whole K range, so split K
    // over a cluster of up to 4 while the clusters still pack into one wave (<= 128 CTAs; a
    // 144-CTA layout of 3-clusters spilled into a second wave).  Graph-timed (scripts/mid_sweep3.py):
    // o M=128 28.4 -> 20.5 us (s4), down M=128 89.5 -> 36.1 (s4), qkv M=128 28.3 -> 23.0 (s2),
    // down M=512 89.3 -> 62.5 (s2)
    const int tiles = n_tiles * m_tiles;
    split = 1;
    for (int k = 4; k >= 2; --k)
      if (tiles * k <= 128) {
        split = k;
        break;
      }
  }
  if (split > KS) split = KS;
  if (split > max_split_for(nt)) split = max_split_for(nt);
  if (split < 1) split = 1;
  c.split = split;
  c.grid_x = n_tiles * split;
  c.grid_y = m_tiles;
  return c;
}

template <int NT, bool BF16, int OUT>
tm_status launch_gemm_t(const CUtensorMap& map, const GemmArgs& args, const Config& c, cudaStream_t stream) {
  auto kern = w4a16_gemm_kernel<NT, BF16, OUT>;
  const int smem = GemmCfg<NT>::smem_bytes(c.split);
  static std::atomic<int> configured[kMaxDevices] = {};  // per instantiation and device
  if (c.split > GemmCfg<NT>::MAX_SPLIT) return TM_ERR_INVALID_ARG;
  tm_status sst = ensure_smem(kern, GemmCfg<NT>::smem_bytes(GemmCfg<NT>::MAX_SPLIT), configured);
  if (sst != TM_OK) return sst;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid_x, c.grid_y, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (c.split > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = c.split;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  CUtensorMap cmap, smap, zmap;
  tm_status cst = out_tensor_map(args.out, args.M, args.N, NT, OUT == OUT_F32 ? 4 : 2, BF16, &cmap);
  if (cst != TM_OK) return cst;
  cst = sz_tensor_map(args.scales, args.K / args.group, args.N, &smap);
  if (cst != TM_OK) return cst;
  cst = sz_tensor_map(args.zeros, args.K / args.group, args.N, &zmap);
  if (cst != TM_OK) return cst;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, map, cmap, smap, zmap, args);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return TM_ERR_CUDA;
  }
  return TM_OK;
}

// caller-owned workspace of tm_gemm_w4a16_ws (null: the library-owned one)
struct UserWs {
  void* ptr;
  int64_t bytes;
};

// grouped (MoE) launch description: expert e's tiles, A/C rows and token count
struct Grouped {
  int E = 0;
  int M_total = 0;
  int tile_start[kMaxExperts + 1] = {};
  int row_start[kMaxExperts] = {};
  int m_count[kMaxExperts] = {};
};

template <int NT, bool BF16, int OUT, bool FS, typename GA = DecNoGroups>
tm_status launch_dec_t(const void* A, const GemmArgs& g, const Config& c, cudaStream_t stream, UserWs ws,
                       const Grouped* grp = nullptr) {
  using Cfg = DecCfg<NT, FS>;
  auto kern = w4a16_dec_kernel<NT, BF16, OUT, FS, GA>;
  static std::atomic<int> configured[kMaxDevices] = {};
  tm_status sst = ensure_smem(kern, Cfg::SMEM, configured);
  if (sst != TM_OK) return sst;
  CUtensorMap ma, ms, mz;
  const int E = grp ? grp->E : 1;
  tm_status st = act_tensor_map_3d(A, g.M, g.a_ks * 64, NT, Cfg::BLOBS, BF16, &ma);
  if (st != TM_OK) return st;
  st = sz_tensor_map(g.scales, E * (g.K / g.group), g.N, &ms);
  if (st != TM_OK) return st;
  st = sz_tensor_map(g.zeros, E * (g.K / g.group), g.N, &mz);
  if (st != TM_OK) return st;
  GA ga{};
  if constexpr (std::is_same<GA, DecGroups>::value) {
    ga.n_experts = grp->E;
    for (int e = 0; e <= grp->E; ++e) ga.tile_start[e] = grp->tile_start[e];
    for (int e = 0; e < grp->E; ++e) {
      ga.row_start[e] = grp->row_start[e];
      ga.m_count[e] = grp->m_count[e];
    }
  }
  DecArgs a;
  a.packed = g.packed;
  a.out = g.out;
  a.M = g.M;
  a.N = g.N;
  a.K = g.K;
  a.group = g.group;
  a.n_tiles = g.N / 128;
  a.m_tiles = (g.M + NT - 1) / NT;
  a.kc = (g.K + Cfg::CH - 1) / Cfg::CH;
  a.total = grp ? static_cast<long long>(grp->tile_start[grp->E]) * a.kc
               : static_cast<long long>(a.m_tiles) * a.n_tiles * a.kc;
  a.trace = g_trace;
  a.cluster = c.kind == 2 ? c.split : 0;
  a.a_ks = g.a_ks;
  if (a.total * static_cast<long long>(c.split) >= (1ll << 32)) return TM_ERR_UNSUPPORTED_SHAPE;  // 32-bit range math
  // stream-K: one partial slot and one flag per CTA (its first segment); the cluster modes
  // reduce in distributed shared memory and need no workspace
  a.counters = nullptr;
  a.workspace = nullptr;
  if (c.kind == 1) {
    st = get_workspace(stream, ws.ptr, ws.bytes, c.split, NT, &a.counters, &a.workspace);
    if (st != TM_OK) return st;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.kind == 2 ? c.grid_x : c.split, 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  cfg.attrs = attrs;
  cfg.numAttrs = 0;
  static const bool no_pdl = std::getenv("TM_NO_PDL") != nullptr;  // experiments only
  if (!no_pdl) {
    attrs[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  if (c.kind == 2 && c.split > 1) {
    attrs[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attrs[cfg.numAttrs].val.clusterDim.x = c.split;
    attrs[cfg.numAttrs].val.clusterDim.y = 1;
    attrs[cfg.numAttrs].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, ms, mz, a, ga);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return TM_ERR_CUDA;
  }
  return TM_OK;
}

template <bool BF16, int OUT>
tm_status launch_sk(const void* A, const GemmArgs& g, const Config& c, cudaStream_t stream, UserWs ws,
                    const Grouped* grp = nullptr) {
  if (grp) {  // grouped (MoE) launches: bf16 in, bf16 out
    if constexpr (BF16 && OUT == OUT_ACT) {
      switch (c.NT) {
        case 16: return launch_dec_t<16, true, OUT_ACT, false, DecGroups>(A, g, c, stream, ws, grp);
        case 32: return launch_dec_t<32, true, OUT_ACT, false, DecGroups>(A, g, c, stream, ws, grp);
        case 64: return launch_dec_t<64, true, OUT_ACT, false, DecGroups>(A, g, c, stream, ws, grp);
      }
    }
    return TM_ERR_INVALID_ARG;
  }
  switch (c.NT) {
    case 16: {
      // fused-scale variant (dequant sets apply the group scales; cluster split-K, group 128):
      // opt-in (TM_FS=1) -- measured 2.5 % slower on the bench mix in its final form
      static const bool fs = std::getenv("TM_FS") != nullptr;
      if (fs && g.group == 128 && c.kind == 2) return launch_dec_t<16, BF16, OUT, true>(A, g, c, stream, ws);
      return launch_dec_t<16, BF16, OUT, false>(A, g, c, stream, ws);
    }
    // (NT = 32/64 keep the scale warps: measured with the fused variant, NT = 32 cluster shapes
    // were 6-13 % slower (2 dequant sets carry the scale work) and NT = 64 spills acc[64])
    case 32: return launch_dec_t<32, BF16, OUT, false>(A, g, c, stream, ws);
    case 64: return launch_dec_t<64, BF16, OUT, false>(A, g, c, stream, ws);
    default: return TM_ERR_INVALID_ARG;
  }
}

template <bool BF16, int OUT>
tm_status launch_gemm(const CUtensorMap& map, const GemmArgs& args, const Config& c, cudaStream_t stream) {
  switch (c.NT) {
    case 16: return launch_gemm_t<16, BF16, OUT>(map, args, c, stream);
    case 32: return launch_gemm_t<32, BF16, OUT>(map, args, c, stream);
    case 64: return launch_gemm_t<64, BF16, OUT>(map, args, c, stream);
    case 128: return launch_gemm_t<128, BF16, OUT>(map, args, c, stream);
    case 256: return launch_gemm_t<256, BF16, OUT>(map, args, c, stream);
    default: return TM_ERR_INVALID_ARG;
  }
}

// CTA-pair prefill (gemm_2sm.cuh): where the tiled kernel would run 128 x 256 tiles without
// split-K, N % 256 == 0, bf16/fp16 output.
template <int NT, bool BF16, int OUT>
tm_status launch_2sm_t(const void* A, const GemmArgs& args, cudaStream_t stream) {
  using Cfg = PairCfg<NT>;
  auto kern = w4a16_gemm_2sm_kernel<NT, BF16, OUT>;
  static std::atomic<int> configured[kMaxDevices] = {};
  tm_status st = ensure_smem(kern, Cfg::SMEM, configured);
  if (st != TM_OK) return st;
  CUtensorMap amap, cmap, smap, zmap;
  st = act_tensor_map(A, args.M, args.a_ks * 64, Cfg::HALF, BF16, &amap);
  if (st != TM_OK) return st;
  st = out_tensor_map(args.out, args.M, args.N, Cfg::NT, OUT == OUT_F32 ? 4 : 2, BF16, &cmap);
  if (st != TM_OK) return st;
  st = sz_tensor_map(args.scales, args.K / args.group, args.N, &smap);
  if (st != TM_OK) return st;
  st = sz_tensor_map(args.zeros, args.K / args.group, args.N, &zmap);
  if (st != TM_OK) return st;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(args.N / 128 * args.split, (args.M + Cfg::NT - 1) / Cfg::NT, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2 * args.split;  // S splits of one CTA pair
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, kern, amap, cmap, smap, zmap, args) != cudaSuccess) {
    (void)cudaGetLastError();
    return TM_ERR_CUDA;
  }
  return TM_OK;
}

template <bool BF16, int OUT>
tm_status launch_2sm(const void* A, const GemmArgs& args, int nt, cudaStream_t stream) {
  if (nt == 64) return launch_2sm_t<64, BF16, OUT>(A, args, stream);
  if (nt == 128) return launch_2sm_t<128, BF16, OUT>(A, args, stream);
  return launch_2sm_t<256, BF16, OUT>(A, args, stream);
}

template <bool BF16>
tm_status launch_pk(const void* A, const GemmArgs& args, const Config& c, cudaStream_t stream) {
  constexpr int NT = kPkNT;
  using Cfg = PkCfg<NT, BF16>;
  auto kern = w4a16_gemm_pk_kernel<NT, BF16>;
  static std::atomic<int> configured[kMaxDevices] = {};
  tm_status st = ensure_smem(kern, Cfg::SMEM, configured);
  if (st != TM_OK) return st;
  CUtensorMap amap, cmap, smap, zmap;
  st = act_tensor_map(A, args.M, args.a_ks * 64, NT, BF16, &amap);
  if (st != TM_OK) return st;
  st = out_tensor_map(args.out, args.M, args.N, NT, 2, BF16, &cmap);
  if (st != TM_OK) return st;
  st = sz_tensor_map(args.scales, args.K / args.group, args.N, &smap);
  if (st != TM_OK) return st;
  st = sz_tensor_map(args.zeros, args.K / args.group, args.N, &zmap);
  if (st != TM_OK) return st;
  const int n_tiles = args.N / 128, m_tiles = (args.M + NT - 1) / NT;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid_x, 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, amap, cmap, smap, zmap, args, n_tiles, m_tiles) != cudaSuccess) {
    (void)cudaGetLastError();
    return TM_ERR_CUDA;
  }
  return TM_OK;
}

template <int NT, int GROUP, bool BF16, int OUT>
tm_status launch_rf_t(const void* A, const GemmArgs& g, const Config& c, cudaStream_t stream, UserWs ws) {
  using Cfg = RfCfg<NT, GROUP>;
  auto kern = w4a16_rf_kernel<NT, GROUP, BF16, OUT>;
  static std::atomic<int> configured[kMaxDevices] = {};
  tm_status st = ensure_smem(kern, Cfg::SMEM, configured);
  if (st != TM_OK) return st;
  CUtensorMap ma, ms, mz;
  st = act_tensor_map_3d(A, g.M, g.a_ks * 64, NT, 4, BF16, &ma);
  if (st != TM_OK) return st;
  st = sz_tensor_map(g.scales, g.K / GROUP, g.N, &ms, Cfg::U);
  if (st != TM_OK) return st;
  st = sz_tensor_map(g.zeros, g.K / GROUP, g.N, &mz, Cfg::U);
  if (st != TM_OK) return st;
  RfArgs a;
  a.packed = g.packed;
  a.out = g.out;
  a.M = g.M;
  a.N = g.N;
  a.K = g.K;
  a.kc = (g.K + 255) / 256;
  const long long T = static_cast<long long>(g.N / 128) * a.kc;
  if (T * c.grid_x >= (1ll << 32)) return TM_ERR_UNSUPPORTED_SHAPE;  // 32-bit range math
  a.total = static_cast<uint32_t>(T);
  a.split = c.split > 0 ? c.split : 0;
  a.a_ks = g.a_ks;
  a.trace = g_trace;
  a.partials = nullptr;
  if (c.split <= 0) {  // stream-K: one partial tile per CTA
    int* flags = nullptr;
    st = get_workspace(stream, ws.ptr, ws.bytes, c.grid_x, NT, &flags, &a.partials, 1);
    if (st != TM_OK) return st;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c.grid_x, 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  cfg.attrs = attrs;
  cfg.numAttrs = 0;
  static const bool no_pdl = std::getenv("TM_NO_PDL") != nullptr;  // experiments only
  if (!no_pdl) {
    attrs[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  if (c.split > 1) {
    attrs[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attrs[cfg.numAttrs].val.clusterDim.x = c.split;
    attrs[cfg.numAttrs].val.clusterDim.y = 1;
    attrs[cfg.numAttrs].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  if (cudaLaunchKernelEx(&cfg, kern, ma, ms, mz, a) != cudaSuccess) {
    (void)cudaGetLastError();
    return TM_ERR_CUDA;
  }
  return TM_OK;
}

template <bool BF16, int OUT>
tm_status launch_rf(const void* A, const GemmArgs& g, const Config& c, cudaStream_t stream, UserWs ws) {
  if (c.NT == 8)
    return g.group == 64 ? launch_rf_t<8, 64, BF16, OUT>(A, g, c, stream, ws)
                         : launch_rf_t<8, 128, BF16, OUT>(A, g, c, stream, ws);
  return g.group == 64 ? launch_rf_t<16, 64, BF16, OUT>(A, g, c, stream, ws)
                       : launch_rf_t<16, 128, BF16, OUT>(A, g, c, stream, ws);
}

// a_K: columns of A (= K, or K / 2 for W8 bit planes: the low planes reuse the activations)
tm_status gemm_common(const void* A, const tm_packed_w4* packed, const void* scales, const void* zeros, void* C,
                      int M, int N, int K, void* stream, bool bf16, int out_kind, UserWs ws = UserWs{nullptr, 0},
                      int a_K = 0) {
  if (a_K == 0) a_K = K;
  if (!packed || !scales || !zeros || !packed->data) return TM_ERR_INVALID_ARG;
  if (M < 0) return TM_ERR_INVALID_ARG;
  const uint32_t want_layout = a_K == K ? TM_LAYOUT_V1 : TM_LAYOUT_V1_W8;
  if (packed->layout != want_layout || packed->K != K || packed->N != N) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(K, N, packed->group);
  if (st != TM_OK) return st;
  if (packed->bytes < static_cast<int64_t>(K) * N / 2) return TM_ERR_INVALID_ARG;
  if (M == 0) return TM_OK;  // no-op; A and C may be empty (null) tensors
  if (!A || !C) return TM_ERR_INVALID_ARG;
  if (!aligned16(A) || !aligned16(packed->data) || !aligned16(scales) || !aligned16(zeros) || !aligned16(C))
    return TM_ERR_MISALIGNED;
  Config c = choose_config(M, N, K);
  if (c.kind == 4 && out_kind == OUT_F32) c = choose_config_tiled(M, N, K);  // fp32 partials: tiled kernel
  GemmArgs args;
  args.packed = static_cast<const uint8_t*>(packed->data);
  args.scales = static_cast<const uint16_t*>(scales);
  args.zeros = static_cast<const uint16_t*>(zeros);
  args.out = C;
  args.M = M;
  args.N = N;
  args.K = K;
  args.group = packed->group;
  args.split = c.split;
  args.a_ks = a_K / 64;
  // raster band: keep band x NT x K x 2 B of activations (<= ~24 MB) L2-resident per band
  {
    const long long per = static_cast<long long>(c.NT) * K * 2;
    long long b = per > 0 ? (24ll << 20) / per : 1;
    if (b < 1) b = 1;
    if (b > 16) b = 16;
    static const int force_band = [] {  // A/B experiments only (1 = the old n-fastest order)
      const char* e = std::getenv("TM_PREFILL_BAND");
      return e ? std::atoi(e) : 0;
    }();
    args.band = force_band > 0 ? force_band : static_cast<int>(b);
  }
  args.trace = g_trace;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c.kind == 4) return bf16 ? launch_pk<true>(A, args, c, s) : launch_pk<false>(A, args, c, s);
  if (c.kind == 3) {
    if (out_kind == OUT_F32) return launch_rf<true, OUT_F32>(A, args, c, s, ws);
    return bf16 ? launch_rf<true, OUT_ACT>(A, args, c, s, ws) : launch_rf<false, OUT_ACT>(A, args, c, s, ws);
  }
  if (c.kind == 1 || c.kind == 2) {
    if (out_kind == OUT_F32) return launch_sk<true, OUT_F32>(A, args, c, s, ws);
    return bf16 ? launch_sk<true, OUT_ACT>(A, args, c, s, ws) : launch_sk<false, OUT_ACT>(A, args, c, s, ws);
  }
  if (c.kind == 5) {
    if (out_kind == OUT_F32) return launch_2sm<true, OUT_F32>(A, args, c.NT, s);
    return bf16 ? launch_2sm<true, OUT_ACT>(A, args, c.NT, s) : launch_2sm<false, OUT_ACT>(A, args, c.NT, s);
  }
  CUtensorMap map;
  st = act_tensor_map(A, M, a_K, c.NT, bf16, &map);
  if (st != TM_OK) return st;
  if (out_kind == OUT_F32) return launch_gemm<true, OUT_F32>(map, args, c, s);
  return bf16 ? launch_gemm<true, OUT_ACT>(map, args, c, s) : launch_gemm<false, OUT_ACT>(map, args, c, s);
}

int aux_grid(long long work, int block) {
  long long g = (work + block - 1) / block;
  const long long cap = static_cast<long long>(num_sms()) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

namespace {
// tokens per attention CTA: split each (sequence, KV head) so the grid holds about two CTAs per
// SM (each CTA streams its tokens through a ring of macro-tiles), at least 128 tokens each
int attn_split_tokens(int B, int Hkv, int Lmax) {
  const long long pairs = static_cast<long long>(B) * Hkv;
  const long long target = 2ll * num_sms();
  long long splits = (target + pairs - 1) / pairs;
  if (splits < 1) splits = 1;
  long long per = (Lmax + splits - 1) / splits;
  per = ((per + kAttnMT - 1) / kAttnMT) * kAttnMT;
  if (per < 128) per = 128;
  if (per > Lmax) per = Lmax;
  return static_cast<int>(per);
}
}  // namespace

namespace {
template <int G, bool BF16>
tm_status launch_attn_t(const CUtensorMap& mk, const CUtensorMap& mv, const AttnArgs& a, cudaStream_t s) {
  auto kern = attn_dec_kernel<G, BF16>;
  static std::atomic<int> configured[kMaxDevices] = {};
  tm_status st = ensure_smem(kern, AttnCfg<G>::SMEM, configured);
  if (st != TM_OK) return st;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.splits, a.Hkv, a.B);
  cfg.blockDim = dim3(kAttnThreads, 1, 1);
  cfg.dynamicSmemBytes = AttnCfg<G>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, mk, mv, a) != cudaSuccess) {
    (void)cudaGetLastError();
    return TM_ERR_CUDA;
  }
  return TM_OK;
}
template <bool BF16>
tm_status launch_attn(int G, const CUtensorMap& mk, const CUtensorMap& mv, const AttnArgs& a, cudaStream_t s) {
  switch (G) {
    case 1: return launch_attn_t<1, BF16>(mk, mv, a, s);
    case 2: return launch_attn_t<2, BF16>(mk, mv, a, s);
    case 4: return launch_attn_t<4, BF16>(mk, mv, a, s);
    case 8: return launch_attn_t<8, BF16>(mk, mv, a, s);
  }
  return TM_ERR_UNSUPPORTED_SHAPE;
}
}  // namespace

extern "C" {

int64_t tm_pack_w4_bytes(int K, int N, int group) {
  const tm_status st = check_shape(K, N, group);
  if (st != TM_OK) return st;
  return static_cast<int64_t>(K) * N / 2;
}

tm_status tm_pack_w4(const uint8_t* q, const void* scales, const void* zeros, int K, int N, int group,
                     tm_packed_w4* packed, void* stream) {
  if (!q || !scales || !zeros || !packed || !packed->data) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(K, N, group);
  if (st != TM_OK) return st;
  if (packed->bytes < static_cast<int64_t>(K) * N / 2) return TM_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(scales) || !aligned16(zeros) || !aligned16(packed->data)) return TM_ERR_MISALIGNED;
  const long long chunks = static_cast<long long>(K) * N / 32;
  pack_w4_kernel<<<aux_grid(chunks, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      q, static_cast<uint4*>(packed->data), K, N);
  // A GEMM reads its weights before griddepcontrol.wait (PDL); the no-op kernel makes sure the
  // GEMM's predecessor is not the kernel that wrote them (it starts after the pack completed).
  noop_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>();
  st = from_cuda(cudaGetLastError());
  if (st != TM_OK) return st;
  packed->K = K;
  packed->N = N;
  packed->group = group;
  packed->layout = TM_LAYOUT_V1;
  return TM_OK;
}

namespace {
tm_status finish_pack(tm_packed_w4* packed, int K, int N, int group, uint32_t layout, cudaStream_t s) {
  noop_kernel<<<1, 32, 0, s>>>();  // the GEMM's predecessor is never the packing kernel (PDL)
  const tm_status st = from_cuda(cudaGetLastError());
  if (st != TM_OK) return st;
  packed->K = K;
  packed->N = N;
  packed->group = group;
  packed->layout = layout;
  return TM_OK;
}
}  // namespace

tm_status tm_pack_awq(const int32_t* qweight, const int32_t* qzeros, int K, int N, int group, tm_packed_w4* packed,
                      void* zeros_out, void* stream) {
  if (!qweight || !qzeros || !packed || !packed->data || !zeros_out) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(K, N, group);
  if (st != TM_OK) return st;
  if (packed->bytes < static_cast<int64_t>(K) * N / 2) return TM_ERR_INVALID_ARG;
  if (!aligned16(qweight) || !aligned16(qzeros) || !aligned16(packed->data) || !aligned16(zeros_out))
    return TM_ERR_MISALIGNED;
  auto s = static_cast<cudaStream_t>(stream);
  const long long chunks = static_cast<long long>(K) * N / 32;
  pack_awq_kernel<<<aux_grid(chunks, 256), 256, 0, s>>>(reinterpret_cast<const uint32_t*>(qweight),
                                                        static_cast<uint4*>(packed->data), K, N);
  const long long nz = static_cast<long long>(K / group) * N;
  unpack_zeros_kernel<<<aux_grid(nz, 256), 256, 0, s>>>(reinterpret_cast<const uint32_t*>(qzeros),
                                                        static_cast<uint16_t*>(zeros_out), nz, N, 1, 0);
  return finish_pack(packed, K, N, group, TM_LAYOUT_V1, s);
}

tm_status tm_pack_gptq(const int32_t* qweight, const int32_t* qzeros, int K, int N, int group, int zero_offset,
                       tm_packed_w4* packed, void* zeros_out, void* stream) {
  if (!qweight || !qzeros || !packed || !packed->data || !zeros_out) return TM_ERR_INVALID_ARG;
  if (zero_offset != 0 && zero_offset != 1) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(K, N, group);
  if (st != TM_OK) return st;
  if (packed->bytes < static_cast<int64_t>(K) * N / 2) return TM_ERR_INVALID_ARG;
  if (!aligned16(qweight) || !aligned16(qzeros) || !aligned16(packed->data) || !aligned16(zeros_out))
    return TM_ERR_MISALIGNED;
  auto s = static_cast<cudaStream_t>(stream);
  const long long chunks = static_cast<long long>(K) * N / 32;
  pack_gptq_kernel<<<aux_grid(chunks, 256), 256, 0, s>>>(reinterpret_cast<const uint32_t*>(qweight),
                                                         static_cast<uint4*>(packed->data), K, N);
  const long long nz = static_cast<long long>(K / group) * N;
  unpack_zeros_kernel<<<aux_grid(nz, 256), 256, 0, s>>>(reinterpret_cast<const uint32_t*>(qzeros),
                                                        static_cast<uint16_t*>(zeros_out), nz, N, 0, zero_offset);
  return finish_pack(packed, K, N, group, TM_LAYOUT_V1, s);
}

int64_t tm_pack_w8_bytes(int K, int N, int group) {
  const tm_status st = check_shape(K, N, group);
  if (st != TM_OK) return st;
  if (K % 256) return TM_ERR_UNSUPPORTED_SHAPE;  // a 256-k decode chunk never straddles the planes
  return static_cast<int64_t>(K) * N;
}

tm_status tm_pack_w8(const uint8_t* q8, const void* scales, const void* zeros8, int K, int N, int group,
                     tm_packed_w4* packed, void* scales_out, void* zeros_out, void* stream) {
  if (!q8 || !scales || !zeros8 || !packed || !packed->data || !scales_out || !zeros_out) return TM_ERR_INVALID_ARG;
  const int64_t need = tm_pack_w8_bytes(K, N, group);
  if (need < 0) return static_cast<tm_status>(need);
  if (packed->bytes < need) return TM_ERR_INVALID_ARG;
  if (!aligned16(q8) || !aligned16(scales) || !aligned16(zeros8) || !aligned16(packed->data) ||
      !aligned16(scales_out) || !aligned16(zeros_out))
    return TM_ERR_MISALIGNED;
  auto s = static_cast<cudaStream_t>(stream);
  const long long chunks = static_cast<long long>(2 * K) * N / 32;
  pack_w8_kernel<<<aux_grid(chunks, 256), 256, 0, s>>>(q8, static_cast<uint4*>(packed->data), K, N);
  const long long nsz = static_cast<long long>(K / group) * N;
  w8_sz_kernel<<<aux_grid(nsz, 256), 256, 0, s>>>(static_cast<const uint16_t*>(scales),
                                                  static_cast<const uint16_t*>(zeros8), static_cast<uint16_t*>(scales_out),
                                                  static_cast<uint16_t*>(zeros_out), nsz);
  return finish_pack(packed, 2 * K, N, group, TM_LAYOUT_V1_W8, s);
}

tm_status tm_gemm_w8a16(const void* A, const tm_packed_w4* packed, const void* scales, const void* zeros, void* C,
                        int M, int N, int K, void* stream) {
  if (K <= 0 || K % 256) return K <= 0 ? TM_ERR_INVALID_ARG : TM_ERR_UNSUPPORTED_SHAPE;
  return gemm_common(A, packed, scales, zeros, C, M, N, 2 * K, stream, true, OUT_ACT, UserWs{nullptr, 0}, K);
}

tm_status tm_unpack_w4(const tm_packed_w4* packed, uint8_t* q_out, void* stream) {
  if (!packed || !packed->data || !q_out) return TM_ERR_INVALID_ARG;
  if (packed->layout != TM_LAYOUT_V1) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(packed->K, packed->N, packed->group);
  if (st != TM_OK) return st;
  if (!aligned16(packed->data)) return TM_ERR_MISALIGNED;
  const long long chunks = static_cast<long long>(packed->K) * packed->N / 32;
  unpack_w4_kernel<<<aux_grid(chunks, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(packed->data), q_out, packed->K, packed->N);
  return from_cuda(cudaGetLastError());
}

tm_status tm_dequant_w4(const tm_packed_w4* packed, const void* scales, const void* zeros, void* W_out, int dtype,
                        void* stream) {
  if (!packed || !packed->data || !scales || !zeros || !W_out) return TM_ERR_INVALID_ARG;
  if (packed->layout != TM_LAYOUT_V1 || (dtype != 0 && dtype != 1)) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(packed->K, packed->N, packed->group);
  if (st != TM_OK) return st;
  if (!aligned16(packed->data) || !aligned16(scales) || !aligned16(zeros)) return TM_ERR_MISALIGNED;
  const long long chunks = static_cast<long long>(packed->K) * packed->N / 32;
  auto s = static_cast<cudaStream_t>(stream);
  const auto in = static_cast<const uint4*>(packed->data);
  const auto sc = static_cast<const uint16_t*>(scales);
  const auto zr = static_cast<const uint16_t*>(zeros);
  auto out = static_cast<uint16_t*>(W_out);
  if (dtype == 0)
    dequant_w4_kernel<true><<<aux_grid(chunks, 256), 256, 0, s>>>(in, sc, zr, out, packed->K, packed->N, packed->group);
  else
    dequant_w4_kernel<false><<<aux_grid(chunks, 256), 256, 0, s>>>(in, sc, zr, out, packed->K, packed->N, packed->group);
  return from_cuda(cudaGetLastError());
}

tm_status tm_debug_dequant_int(const tm_packed_w4* packed, const void* zeros, void* W_out, int dtype, void* stream) {
  if (!packed || !packed->data || !zeros || !W_out) return TM_ERR_INVALID_ARG;
  if (packed->layout != TM_LAYOUT_V1 || (dtype != 0 && dtype != 1)) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(packed->K, packed->N, packed->group);
  if (st != TM_OK) return st;
  if (!aligned16(packed->data) || !aligned16(zeros)) return TM_ERR_MISALIGNED;
  const long long chunks = static_cast<long long>(packed->K) * packed->N / 32;
  auto s = static_cast<cudaStream_t>(stream);
  const auto in = static_cast<const uint4*>(packed->data);
  const auto zr = static_cast<const uint16_t*>(zeros);
  auto out = static_cast<uint16_t*>(W_out);
  if (dtype == 0)
    dequant_int_kernel<true><<<aux_grid(chunks, 256), 256, 0, s>>>(in, zr, out, packed->K, packed->N, packed->group);
  else
    dequant_int_kernel<false><<<aux_grid(chunks, 256), 256, 0, s>>>(in, zr, out, packed->K, packed->N, packed->group);
  return from_cuda(cudaGetLastError());
}

tm_status tm_gemm_w4a16(const void* A, const tm_packed_w4* packed, const void* scales, const void* zeros, void* C,
                        int M, int N, int K, void* stream) {
  return gemm_common(A, packed, scales, zeros, C, M, N, K, stream, true, OUT_ACT);
}

tm_status tm_gemm_w4a16_f16(const void* A, const tm_packed_w4* packed, const void* scales, const void* zeros, void* C,
                            int M, int N, int K, void* stream) {
  return gemm_common(A, packed, scales, zeros, C, M, N, K, stream, false, OUT_ACT);
}

tm_status tm_gemm_w4a16_partial_f32(const void* A, const tm_packed_w4* packed, const void* scales,
                                    const void* zeros, float* C_partial, int M, int N, int K, void* stream) {
  return gemm_common(A, packed, scales, zeros, C_partial, M, N, K, stream, true, OUT_F32);
}

int64_t tm_gemm_workspace_bytes(int M, int N, int K, int group) {
  if (M < 0) return TM_ERR_INVALID_ARG;
  const tm_status st = check_shape(K, N, group);
  if (st != TM_OK) return st;
  if (M == 0) return 0;
  const Config c = choose_config(M, N, K);
  if (c.kind == 3) {  // register-fed decode: stream-K mode needs [P][2] partial tiles + tile counters
    if (c.split > 0) return 0;
    return static_cast<int64_t>(ws_flag_bytes(c.grid_x) + static_cast<size_t>(c.grid_x) * c.NT * 128 * sizeof(float));
  }
  if (c.kind != 1) return 0;
  return static_cast<int64_t>(ws_flag_bytes(c.split) + static_cast<size_t>(c.split) * c.NT * 128 * sizeof(float));
}

tm_status tm_gemm_w4a16_ws(const void* A, const tm_packed_w4* packed, const void* scales, const void* zeros, void* C,
                           int M, int N, int K, int a_dtype, int c_dtype, void* workspace, int64_t workspace_bytes,
                           void* stream) {
  if (a_dtype != TM_DTYPE_BF16 && a_dtype != TM_DTYPE_FP16) return TM_ERR_INVALID_ARG;
  if (c_dtype != a_dtype && !(c_dtype == TM_DTYPE_F32 && a_dtype == TM_DTYPE_BF16)) return TM_ERR_INVALID_ARG;
  if (workspace_bytes < 0 || (workspace == nullptr && workspace_bytes != 0)) return TM_ERR_INVALID_ARG;
  if (M > 0 && workspace == nullptr) {
    const int64_t need = tm_gemm_workspace_bytes(M, N, K, packed ? packed->group : 0);
    if (need > 0) return TM_ERR_INVALID_ARG;  // this shape needs a workspace
  }
  return gemm_common(A, packed, scales, zeros, C, M, N, K, stream, a_dtype == TM_DTYPE_BF16,
                     c_dtype == TM_DTYPE_F32 ? OUT_F32 : OUT_ACT, UserWs{workspace, workspace_bytes});
}

tm_status tm_gemm_w4a16_grouped(const void* A, const tm_packed_w4* packed, const void* scales, const void* zeros,
                                void* C, const int32_t* m_per_expert, int n_experts, int N, int K, void* stream) {
  if (!packed || !packed->data || !scales || !zeros || !m_per_expert) return TM_ERR_INVALID_ARG;
  if (n_experts < 1 || n_experts > kMaxExperts) return TM_ERR_UNSUPPORTED_SHAPE;
  if (packed->layout != TM_LAYOUT_V1 || packed->K != K || packed->N != N) return TM_ERR_INVALID_ARG;
  tm_status st = check_shape(K, N, packed->group);
  if (st != TM_OK) return st;
  if (packed->bytes < static_cast<int64_t>(n_experts) * K * N / 2) return TM_ERR_INVALID_ARG;
  Grouped grp;
  grp.E = n_experts;
  int max_m = 0;
  for (int e = 0; e < n_experts; ++e) {
    if (m_per_expert[e] < 0) return TM_ERR_INVALID_ARG;
    grp.row_start[e] = grp.M_total;
    grp.m_count[e] = m_per_expert[e];
    grp.M_total += m_per_expert[e];
    if (m_per_expert[e] > max_m) max_m = m_per_expert[e];
  }
  if (grp.M_total == 0) return TM_OK;  // no tokens routed: nothing to do
  if (!A || !C) return TM_ERR_INVALID_ARG;
  if (!aligned16(A) || !aligned16(packed->data) || !aligned16(scales) || !aligned16(zeros) || !aligned16(C))
    return TM_ERR_MISALIGNED;
  const int nt = max_m <= 16 ? 16 : (max_m <= 32 ? 32 : 64);
  const int n_tiles = N / 128;
  for (int e = 0; e < n_experts; ++e)  // experts with no tokens get no tiles (their weights stay unread)
    grp.tile_start[e + 1] = grp.tile_start[e] + ((grp.m_count[e] + nt - 1) / nt) * n_tiles;
  const Config c = decode_config(nt, grp.tile_start[n_experts], K);
  GemmArgs args;
  args.packed = static_cast<const uint8_t*>(packed->data);
  args.scales = static_cast<const uint16_t*>(scales);
  args.zeros = static_cast<const uint16_t*>(zeros);
  args.out = C;
  args.M = grp.M_total;
  args.N = N;
  args.K = K;
  args.group = packed->group;
  args.split = c.split;
  args.band = 1;
  args.a_ks = K / 64;
  args.trace = g_trace;
  return launch_sk<true, OUT_ACT>(A, args, c, static_cast<cudaStream_t>(stream), UserWs{nullptr, 0}, &grp);
}

int64_t tm_attn_workspace_bytes(int B, int Hq, int Hkv, int Lmax) {
  if (B <= 0 || Hq <= 0 || Hkv <= 0 || Lmax <= 0 || Hq % Hkv) return TM_ERR_INVALID_ARG;
  const int G = Hq / Hkv;
  if ((G & (G - 1)) || G > 8 || Lmax % kAttnMT) return TM_ERR_UNSUPPORTED_SHAPE;
  const long long splits = (Lmax + attn_split_tokens(B, Hkv, Lmax) - 1) / attn_split_tokens(B, Hkv, Lmax);
  if (splits == 1) return 0;
  return static_cast<int64_t>(ws_flag_bytes(B * Hkv)) + static_cast<int64_t>(B) * Hkv * splits * G * (kAttnD + 2) * 4;
}


tm_status tm_attn_decode_kv8(const void* Q, const void* k_codes, const void* v_codes, const void* k_sz,
                             const void* v_sz, const int32_t* seq_lens, void* O, int B, int Hq, int Hkv, int Lmax,
                             float softmax_scale, int q_dtype, void* workspace, int64_t workspace_bytes,
                             void* stream) {
  if (!Q || !k_codes || !v_codes || !k_sz || !v_sz || !seq_lens || !O) return TM_ERR_INVALID_ARG;
  if (q_dtype != TM_DTYPE_BF16 && q_dtype != TM_DTYPE_FP16) return TM_ERR_INVALID_ARG;
  const int64_t need = tm_attn_workspace_bytes(B, Hq, Hkv, Lmax);
  if (need < 0) return static_cast<tm_status>(need);
  if (need > 0 && (!workspace || workspace_bytes < need)) return TM_ERR_INVALID_ARG;
  if (!aligned16(Q) || !aligned16(k_codes) || !aligned16(v_codes) || !aligned16(k_sz) || !aligned16(v_sz) ||
      !aligned16(O) || (workspace && !aligned16(workspace)))
    return TM_ERR_MISALIGNED;
  const long long rows = static_cast<long long>(B) * Hkv * Lmax;
  if (rows >= (1ll << 31)) return TM_ERR_UNSUPPORTED_SHAPE;
  CUtensorMap mk, mv;
  tm_status st = kv_tensor_map(k_codes, rows, &mk);
  if (st != TM_OK) return st;
  st = kv_tensor_map(v_codes, rows, &mv);
  if (st != TM_OK) return st;
  AttnArgs a;
  a.q = static_cast<const uint16_t*>(Q);
  a.ksz = static_cast<const uint32_t*>(k_sz);
  a.vsz = static_cast<const uint32_t*>(v_sz);
  a.seq_lens = seq_lens;
  a.out = static_cast<uint16_t*>(O);
  a.B = B;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.Lmax = Lmax;
  a.split_tokens = attn_split_tokens(B, Hkv, Lmax);
  a.splits = (Lmax + a.split_tokens - 1) / a.split_tokens;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  a.counters = need > 0 ? static_cast<int*>(workspace) : nullptr;
  a.part = need > 0 ? reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + ws_flag_bytes(B * Hkv)) : nullptr;
  const int G = Hq / Hkv;
  auto s = static_cast<cudaStream_t>(stream);
  return q_dtype == TM_DTYPE_BF16 ? launch_attn<true>(G, mk, mv, a, s) : launch_attn<false>(G, mk, mv, a, s);
}

tm_status tm_tp_finalize(const float* in_f32, void* out_bf16, int64_t count, void* stream) {
  if (!in_f32 || !out_bf16 || count < 0) return TM_ERR_INVALID_ARG;
  if (!aligned16(in_f32) || !aligned16(out_bf16)) return TM_ERR_MISALIGNED;
  if (count == 0) return TM_OK;
  auto s = static_cast<cudaStream_t>(stream);
  const long long n4 = count / 4;
  if (n4 > 0)
    tp_finalize_kernel<<<aux_grid(n4, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(in_f32),
                                                          static_cast<uint2*>(out_bf16), n4);
  const long long tail = count - n4 * 4;
  if (tail > 0)
    tp_finalize_tail_kernel<<<1, 32, 0, s>>>(in_f32, static_cast<__nv_bfloat16*>(out_bf16), n4 * 4, count);
  return from_cuda(cudaGetLastError());
}

tm_status tm_tp_allreduce_finalize(const float* const* partials, uint32_t* const* signals, const float* multicast,
                                   int rank, int world, int64_t count, void* out_bf16, void* stream) {
  if (!partials || !signals || !out_bf16 || count < 0) return TM_ERR_INVALID_ARG;
  if (world < 1 || world > kTpMaxRanks || rank < 0 || rank >= world) return TM_ERR_INVALID_ARG;
  TpReduceArgs a{};
  for (int r = 0; r < world; ++r) {
    if (!partials[r] || !signals[r]) return TM_ERR_INVALID_ARG;
    if (!aligned16(partials[r]) || (reinterpret_cast<uintptr_t>(signals[r]) & 3)) return TM_ERR_MISALIGNED;
    a.partials[r] = partials[r];
    a.signals[r] = signals[r];
  }
  if (!aligned16(out_bf16) || (multicast && !aligned16(multicast))) return TM_ERR_MISALIGNED;
  a.multicast = multicast;
  a.out = static_cast<__nv_bfloat16*>(out_bf16);
  a.count = count;
  a.rank = rank;
  a.world = world;
  // every rank runs the barriers, also for count == 0 (peers may have work)
  tp_allreduce_finalize_kernel<<<kTpBlocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return from_cuda(cudaGetLastError());
}

tm_status tm_set_gemm_override(int tile_m, int split_k) {
  if (tile_m > 0 && tile_m != 16 && tile_m != 32 && tile_m != 64 && tile_m != 128 && tile_m != 256)
    return TM_ERR_INVALID_ARG;
  if (split_k > 8 || (split_k > 0 && tile_m > 0 && split_k > max_split_for(tile_m))) return TM_ERR_INVALID_ARG;
  if (split_k < -4096) return TM_ERR_INVALID_ARG;
  if (split_k < 0 && tile_m > 64) return TM_ERR_INVALID_ARG;  // stream-K is the decode kernel (tile_m <= 64)
  g_override_tile.store(tile_m > 0 ? tile_m : 0);
  g_override_split.store(split_k);
  return TM_OK;
}

tm_status tm_query_gemm_config(int M, int N, int K, int* tile_m, int* split_k, int* grid_ctas) {
  if (M <= 0 || N <= 0 || K <= 0 || N % 128 || K % 64) return TM_ERR_INVALID_ARG;
  const Config c = choose_config(M, N, K);
  if (tile_m) *tile_m = c.NT;
  if (split_k) *split_k = c.split;
  if (grid_ctas) *grid_ctas = c.grid_x * c.grid_y;
  if (split_k && c.kind == 1) *split_k = -c.split;  // negative: persistent stream-K CTA count
  return TM_OK;
}

tm_status tm_query_gemm_kind(int M, int N, int K, int* kind) {
  if (M <= 0 || N <= 0 || K <= 0 || N % 128 || K % 64 || !kind) return TM_ERR_INVALID_ARG;
  *kind = choose_config(M, N, K).kind;
  return TM_OK;
}

tm_status tm_set_prefill_persistent(int on) {
  g_pk.store(on ? 1 : 0);
  return TM_OK;
}

tm_status tm_set_prefill_pair(int on) {
  if (on < 0 || on > 3) return TM_ERR_INVALID_ARG;
  g_pair.store(on == 3 ? 1 : on);
  g_pair128.store(on == 3 ? 0 : 1);
  return TM_OK;
}

tm_status tm_set_decode_path(int path, int split) {
  if (path < 0 || path > 2 || split > 8 || split < -4096) return TM_ERR_INVALID_ARG;
  g_dec_path.store(path);
  g_rf_split.store(split);
  return TM_OK;
}

tm_status tm_set_decode_cluster(int cs) {
  if (cs < -1 || cs > 8) return TM_ERR_INVALID_ARG;
  g_dec_cluster.store(cs);
  return TM_OK;
}

const char* tm_status_string(tm_status s) {
  switch (s) {
    case TM_OK: return "TM_OK";
    case TM_ERR_INVALID_ARG: return "TM_ERR_INVALID_ARG";
    case TM_ERR_UNSUPPORTED_SHAPE: return "TM_ERR_UNSUPPORTED_SHAPE";
    case TM_ERR_MISALIGNED: return "TM_ERR_MISALIGNED";
    case TM_ERR_CUDA: return "TM_ERR_CUDA";
    case TM_ERR_NO_DEVICE: return "TM_ERR_NO_DEVICE";
  }
  return "TM_ERR_UNKNOWN";
}

tm_status tm_set_trace(void* buf, int64_t bytes) {
  if (buf && bytes < 4) return TM_ERR_INVALID_ARG;
  g_trace = static_cast<uint32_t*>(buf);
  return TM_OK;
}

const char* tm_version(void) { return "tm_w4a16 0.1 (sm_100a, LAYOUT v1)"; }

}  // extern "C"
