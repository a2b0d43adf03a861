// host.cuh -- host-side helpers shared by the ABI translation unit (santa_abi.cu) and the
// per-(family, dtype, head_dim) kernel-instantiation units (inst.cu): workspace layout, launch
// helpers, per-device attribute caches, tensor-map encoding, and the launcher declarations.
#pragma once
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include <cudaTypedefs.h>

#include "bernoulli_kernels.cuh"
#include "bern_tma_kernel.cuh"
#include "common.cuh"
#include "dense_kernels.cuh"
#include "dense_stream_kernel.cuh"
#include "flash_kernels.cuh"
#include "philox.cuh"
#include "prop_kernels.cuh"
#include "sample_kernels.cuh"
#include "sample_fast.cuh"
#include "score_kernels.cuh"
#include "step_kernel.cuh"
#include "step_tc_kernel.cuh"

namespace santa_host {
using namespace santa;



// Decode paths: the pipelined single-launch step kernel (step_kernel.cuh; default when eligible)
// and the score pass + PDL-chained sampler pair (fp32 caches, page sizes not a multiple of 64,
// contexts > 64k, profiling, and the sequence-sharded phases).

constexpr int kTcMinHeads = 1024;  // AUTO runs the tcgen05 step kernel from here (and S <= 256)

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct WsLayout {
  int L = 64, Cmax = 0, Cmax256 = 0;
  size_t stash = 0, cstats = 0, tickets = 0, flags = 0, sync = 0, bern = 0, bfrag = 0, total = 0;
  size_t step_rec = 0, step_stash = 0, step_part = 0;  // step kernel's tagged regions
  size_t dense_o = 0, dense_ml = 0;  // dense_split_kernel partials
};

constexpr int kMaxSeqlen = 1 << 20;   // chunk-CDF tables are sized for <= 8192 chunks of <= 128 keys

inline int elem_bytes(int dtype) { return dtype == SANTA_F32 ? 4 : 2; }

inline santa_status validate_geometry(const santa_geometry* g) {
  if (!g) return SANTA_ERR_INVALID_ARG;
  if (g->batch < 1 || g->n_heads < 1 || g->n_kv_heads < 1) return SANTA_ERR_SHAPE;
  if (g->n_heads % g->n_kv_heads != 0) return SANTA_ERR_SHAPE;
  const int G = g->n_heads / g->n_kv_heads;
  if (!(G == 1 || G == 2 || G == 4 || G == 8)) return SANTA_ERR_UNSUPPORTED;
  if (g->head_dim != 64 && g->head_dim != 128) return SANTA_ERR_UNSUPPORTED;
  if (g->dtype != SANTA_BF16 && g->dtype != SANTA_F32 && g->dtype != SANTA_F16) return SANTA_ERR_INVALID_ARG;
  if (g->max_seqlen < 1) return SANTA_ERR_EMPTY_DISTRIBUTION;
  if (g->max_seqlen > kMaxSeqlen) return SANTA_ERR_UNSUPPORTED;
  if (!(g->scale >= 0.f) || !std::isfinite(g->scale)) return SANTA_ERR_INVALID_ARG;
  if (g->batch_offset < 0 || g->head_offset < 0) return SANTA_ERR_INVALID_ARG;
  if (g->page_table) {
    if (g->page_size < 16 || g->page_size % 16 != 0) return SANTA_ERR_SHAPE;
    if (g->max_pages_per_seq < (g->max_seqlen + g->page_size - 1) / g->page_size) return SANTA_ERR_SHAPE;
    if (!aligned16(g->page_table) && (reinterpret_cast<uintptr_t>(g->page_table) & 3u)) return SANTA_ERR_ALIGNMENT;
  }
  return SANTA_OK;
}

inline WsLayout layout(const santa_geometry* g, int S) {
  WsLayout L;
  const int G = g->n_heads / g->n_kv_heads;
  const size_t B = g->batch, H = g->n_heads, Hkv = g->n_kv_heads, D = g->head_dim;
  // SANTA chunk length: 64 keys (the fast register epilogue and ballot search) up to 8192 chunks
  // per sequence (512k tokens: the sampler's fp64 chunk-CDF tables take 16 B per chunk of shared
  // memory); longer contexts double L until <= 8192 chunks
  L.L = 64;
  while ((g->max_seqlen + L.L - 1) / L.L > 8192) L.L *= 2;
  L.Cmax = (g->max_seqlen + L.L - 1) / L.L;
  L.Cmax256 = (g->max_seqlen + 255) / 256;  // dense reference / Bernoulli chunking
  size_t off = 0;
  L.flags = off; off = align256(off + 4);     // flag word at offset 0 (santa_read_error_flags)
  L.tickets = off; off = align256(off + B * Hkv * 4);  // S-independent offset (seq-shard phases)
  // step-kernel words: epoch, exit_ticket, head_ticket [B*H] (tickets zero at rest; the epoch
  // advances once per launch).  S-independent offset.
  L.sync = off; off = align256(off + (2 + B * H) * 4);
  const size_t keys = (size_t)L.Cmax * L.L > (size_t)L.Cmax256 * 256 ? (size_t)L.Cmax * L.L : (size_t)L.Cmax256 * 256;
  const size_t stash_bytes = B * H * keys * 4;
  const size_t opart_bytes = B * H * (size_t)L.Cmax256 * D * 4;   // dense partials share this region
  L.stash = off; off = align256(off + (stash_bytes > opart_bytes ? stash_bytes : opart_bytes));
  const size_t cmx = L.Cmax > L.Cmax256 ? L.Cmax : L.Cmax256;
  L.cstats = off; off = align256(off + B * H * cmx * 8);
  L.bern = off; off = align256(off + B * Hkv * ((size_t)G * D * 4 + D * 4 + 256));  // weights, sel, sel_n
  L.bfrag = off; off = align256(off + B * Hkv * (size_t)(D / 16) * 96 * 8);  // bern_tma_kernel B fragments
  // step kernel: tagged chunk records, tagged fixed-point stash, tagged split partials (separate
  // from the two-kernel path's untagged regions so the paths can share one workspace)
  L.step_rec = off; off = align256(off + B * H * (size_t)L.Cmax * 16);
  L.step_stash = off; off = align256(off + B * H * (size_t)L.Cmax * 64 * 4);
  L.step_part = off; off = align256(off + B * H * (size_t)kStepMaxSplits * D * 8);
  const size_t dslots = ((size_t)kDenseSplitMaxCtas + B * Hkv) * kDenseWarpsMax;  // dense_split_kernel slots
  L.dense_o = off; off = align256(off + dslots * G * D * 4);
  L.dense_ml = off; off = align256(off + dslots * G * 8);
  L.total = off;
  return L;
}

inline santa_status check_ws(const santa_geometry* g, int S, void* ws, size_t ws_bytes, WsLayout* L) {
  *L = layout(g, S);
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255u)) return SANTA_ERR_WORKSPACE;
  if (ws_bytes < L->total) return SANTA_ERR_WORKSPACE;
  return SANTA_OK;
}

template <typename P>
P* at(void* ws, size_t off) { return reinterpret_cast<P*>(reinterpret_cast<char*>(ws) + off); }

inline KvLayout kv_layout(const santa_geometry* g) {
  KvLayout kv;
  kv.page_table = g->page_table;
  kv.page_size = g->page_table ? g->page_size : g->max_seqlen;
  kv.max_pages = g->page_table ? g->max_pages_per_seq : 1;
  kv.n_kv_heads = g->n_kv_heads;
  kv.page_shift = -1;
  if (g->page_table && (g->page_size & (g->page_size - 1)) == 0) {
    int s = 0;
    while ((1 << s) < g->page_size) ++s;
    kv.page_shift = s;
  }
  return kv;
}

inline float scale_log2(const santa_geometry* g) {
  const float s = g->scale > 0.f ? g->scale : 1.0f / std::sqrt((float)g->head_dim);
  return s * kLog2e;
}

inline santa_status last_cuda() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return SANTA_ERR_CUDA;
  }
  return SANTA_OK;
}

template <typename Kern, typename... Args>
cudaError_t launch(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---- dispatch helpers -----------------------------------------------------------------
template <template <typename, int, int> class F, typename... A>
inline santa_status dispatch(int dtype, int D, int G, A&&... a) {
#define SANTA_G(T, DD)                                        \
  switch (G) {                                                \
    case 1: return F<T, DD, 1>::run(a...);                    \
    case 2: return F<T, DD, 2>::run(a...);                    \
    case 4: return F<T, DD, 4>::run(a...);                    \
    case 8: return F<T, DD, 8>::run(a...);                    \
    default: return SANTA_ERR_UNSUPPORTED;                    \
  }
#define SANTA_D(T)                                            \
  if (D == 64) { SANTA_G(T, 64) } else { SANTA_G(T, 128) }
  if (dtype == SANTA_BF16) { SANTA_D(__nv_bfloat16) }
  if (dtype == SANTA_F16) { SANTA_D(__half) }
  if (dtype == SANTA_F32) { SANTA_D(float) }
#undef SANTA_D
#undef SANTA_G
  return SANTA_ERR_UNSUPPORTED;
}

struct DecodeArgs {
  const santa_geometry* g;
  const void *q, *K, *V;
  const int32_t* seqlens;
  int S, mode;
  uint64_t seed, offset;
  void* out;
  float* out_f32;
  int32_t* idx_out;
  void* ws;
  WsLayout L;
  cudaStream_t st;
  cudaEvent_t const* events;  // NULL or [3]
  // seq-shard
  const double* stats_all;
  int rank, world;
  const int32_t* token_offset;
  int Lc = 0, Cc = 0;         // chunking the sampler reads (0 => the SANTA layout L / Cmax)
  bool tensor_core = false;   // step kernel: score stage on tcgen05 (step_tc_kernel.cuh)
  const void* k_new = nullptr;  // fused KV append (two-kernel path's score pass)
  const void* v_new = nullptr;
  void* K_w = nullptr;
  void* V_w = nullptr;
};

// ---- host-side caches: per device, safe under concurrent calls from several host threads ----
// (santa.h promises reentrancy: the only process-wide state is these caches of facts about the
// device and the kernels, each written idempotently.)
constexpr int kMaxDevices = 64;

inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev;
}

inline int num_sms() {
  static std::atomic<int> cached[kMaxDevices];  // zero-initialised (static storage)
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return 148;
  int n = cached[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    cached[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per (kernel, device): remember the largest
// value set for each pair.  Two threads racing on a first call both set the attribute (idempotent).
inline std::mutex g_attr_mu;

template <typename Kern>
cudaError_t ensure_smem(Kern kern, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  static std::map<std::pair<const void*, int>, size_t> cache;  // guarded by g_attr_mu
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), current_device());
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = cache.find(key);
    if (it != cache.end() && it->second >= smem) return cudaSuccess;
  }
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  size_t& v = cache[key];
  if (v < smem) v = smem;
  return cudaSuccess;
}

// Can a persistent kernel keep one CTA per SM at this block size and smem?  Cached per (kernel,
// device, smem): the host-side cost per call matters at ~15-25 us per step.
template <typename Kern>
inline bool fits_one_per_sm(Kern kern, int nthreads, size_t smem) {
  static std::map<std::pair<std::pair<const void*, int>, size_t>, bool> cache;  // guarded by g_attr_mu
  const auto key = std::make_pair(std::make_pair(reinterpret_cast<const void*>(kern), current_device()), smem);
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int occ = 0;
  const bool r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nthreads, smem) == cudaSuccess && occ >= 1;
  if (!r) cudaGetLastError();
  std::lock_guard<std::mutex> lk(g_attr_mu);
  cache[key] = r;
  return r;
}

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
    return nullptr;
  }();  // C++11 function-local static: initialised once, thread-safe
  return fn;
}

// K viewed as a 2-D tensor [rows][D] (D contiguous); 64 x 64-element boxes, 128B swizzle.
// The encoded descriptor depends only on (address, rows, D, dtype, box): a small per-thread cache of
// the last encodings (no lock; a decode loop re-encodes nothing -- cuTensorMapEncodeTiled is ~1 us of
// host time per call, on the critical path when steps are launched back to back).
struct KmapKey {
  const void* K;
  uint64_t rows;
  int D, dtype, box_rows;
  bool operator==(const KmapKey& o) const {
    return K == o.K && rows == o.rows && D == o.D && dtype == o.dtype && box_rows == o.box_rows;
  }
};
inline bool make_kmap_uncached(CUtensorMap* m, const void* K, uint64_t rows, int D, int dtype, int box_rows);
inline bool make_kmap(CUtensorMap* m, const void* K, uint64_t rows, int D, int dtype, int box_rows = 64) {
  constexpr int kSlots = 16;
  thread_local KmapKey keys[kSlots] = {};
  thread_local CUtensorMap maps[kSlots];
  thread_local int next = 0;
  const KmapKey key{K, rows, D, dtype, box_rows};
  for (int i = 0; i < kSlots; ++i)
    if (keys[i] == key) {
      *m = maps[i];
      return true;
    }
  if (!make_kmap_uncached(m, K, rows, D, dtype, box_rows)) return false;
  keys[next] = key;
  maps[next] = *m;
  next = (next + 1) % kSlots;
  return true;
}
inline bool make_kmap_uncached(CUtensorMap* m, const void* K, uint64_t rows, int D, int dtype, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, dtype == SANTA_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
            const_cast<void*>(K), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// q viewed as [B*H rows][D]; boxes of G rows x 64 elements, 128B swizzle (the tcgen05 B operand).
inline bool make_qmap(CUtensorMap* m, const void* q, uint64_t rows, int D, int dtype, int G) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)G};
  cuuint32_t es[2] = {1, 1};
  return fn(m, dtype == SANTA_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
            const_cast<void*>(q), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline ScoreParams make_score_params(const DecodeArgs& a) {
  ScoreParams p = {};
  p.q = a.q;
  p.K = a.K;
  p.kv = kv_layout(a.g);
  p.seqlens = a.seqlens;
  p.B = a.g->batch;
  p.H = a.g->n_heads;
  p.Hkv = a.g->n_kv_heads;
  p.scale_log2 = scale_log2(a.g);
  p.stash = at<float>(a.ws, a.L.stash);
  p.cstats = at<float2>(a.ws, a.L.cstats);
  p.Cmax = a.L.Cmax;
  p.L = a.L.L;
  p.stash_stride = a.L.Cmax * a.L.L;
  p.tickets = at<uint32_t>(a.ws, a.L.tickets);
  p.flags = at<uint32_t>(a.ws, a.L.flags);
  return p;
}

inline bool stream_eligible(const santa_geometry* g) {
  return g->dtype != SANTA_F32 && (!g->page_table || g->page_size % kStageKeys == 0);
}

inline SampleParams make_sample_params(const DecodeArgs& a) {
  SampleParams p = {};
  p.stash = at<float>(a.ws, a.L.stash);
  p.cstats = at<float2>(a.ws, a.L.cstats);
  p.Cmax = a.Cc ? a.Cc : a.L.Cmax;
  p.L = a.Lc ? a.Lc : a.L.L;
  p.stash_stride = p.Cmax * p.L;
  p.V = a.V;
  p.kv = kv_layout(a.g);
  p.seqlens = a.seqlens;
  p.B = a.g->batch;
  p.H = a.g->n_heads;
  p.Hkv = a.g->n_kv_heads;
  p.S = a.S;
  p.mode = a.mode;
  p.seed = a.seed;
  p.offset = a.offset;
  p.batch_offset = a.g->batch_offset;
  p.head_offset = a.g->head_offset;
  p.out = a.out;
  p.out_f32 = a.out_f32;
  p.idx_out = a.idx_out;
  p.flags = at<uint32_t>(a.ws, a.L.flags);
  p.stats_all = a.stats_all;
  p.rank = a.rank;
  p.world = a.world;
  p.token_offset = a.token_offset;
  p.split_partial = nullptr;
  // tools only (tools/sample_trace.py): SANTA_SAMPLE_TRACE=<device address> of a [B*H][16] u64 buffer
  // receives the sampler's per-phase globaltimer stamps; unset in every library use
  static const unsigned long long trace_addr =
      std::getenv("SANTA_SAMPLE_TRACE") ? std::strtoull(std::getenv("SANTA_SAMPLE_TRACE"), nullptr, 0) : 0ull;
  p.trace = reinterpret_cast<unsigned long long*>(trace_addr);
  p.cluster = 1;
  return p;
}

// The whole step in one pipelined cooperative launch (step_kernel.cuh).  Returns
// SANTA_ERR_UNSUPPORTED (nothing launched) when the configuration does not qualify, in which
// case the caller runs the two-kernel path.
// A cooperative launch the device cannot co-schedule (e.g. SMs held by another context) is
// "unsupported here", not a failure: AUTO then runs the two-kernel path.
inline santa_status coop_status(cudaError_t e) {
  if (e == cudaSuccess) return SANTA_OK;
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();  // clear the sticky-free launch error
    return SANTA_ERR_UNSUPPORTED;
  }
  return SANTA_ERR_CUDA;
}

inline StepSync make_step_sync(const DecodeArgs& a) {
  StepSync sy;
  uint32_t* base = at<uint32_t>(a.ws, a.L.sync);
  sy.epoch = base;
  sy.exit_ticket = base + 1;
  sy.head_ticket = base + 2;
  sy.rec = at<ulonglong2>(a.ws, a.L.step_rec);
  sy.stash = at<uint32_t>(a.ws, a.L.step_stash);
  sy.part = at<unsigned long long>(a.ws, a.L.step_part);
  sy.trace = nullptr;
  return sy;
}

// ---- launchers: one template per kernel family; run() is defined in runners.cuh and explicitly
// instantiated per (dtype, head_dim) in inst.cu, so the kernels compile in parallel units ----
template <typename T, int D, int G>
struct RunScore { static santa_status run(const DecodeArgs& a); };
template <typename T, int D, int G>
struct RunSample { static santa_status run(const DecodeArgs& a); };
template <typename T, int D, int G>
struct RunProp { static santa_status run(const DecodeArgs& a); };
template <typename T, int D, int G>
struct RunFlash { static santa_status run(const DecodeArgs& a, int cpt, int mmax); };
template <typename T, int D, int G>
struct RunStep {
  static santa_status run_tc(const DecodeArgs& a, const ScoreParams& sp, const SampleParams& pp, int CS, int grid);
  static santa_status run(const DecodeArgs& a);
};
template <typename T, int D, int G>
struct RunDense { static santa_status run(const DecodeArgs& a); };
template <typename T, int D, int G>
struct RunBern {
  static santa_status run(const DecodeArgs& a, const void* Kt, int nB, int stratified, int mean_group,
                          float* scores, uint8_t* mask, bool for_decode);
};

}  // namespace santa_host
