// santa_abi.cu -- host side of libsanta.so: argument validation, workspace layout,
// template dispatch and (PDL-chained) launches.  See include/santa.h for the contract.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include <cudaTypedefs.h>

#include "bernoulli_kernels.cuh"
#include "common.cuh"
#include "dense_kernels.cuh"
#include "dense_stream_kernel.cuh"
#include "flash_kernels.cuh"
#include "philox.cuh"
#include "prop_kernels.cuh"
#include "sample_kernels.cuh"
#include "score_kernels.cuh"
#include "step_kernel.cuh"
#include "step_tc_kernel.cuh"

using namespace santa;

namespace {


// Decode paths: the pipelined single-launch step kernel (step_kernel.cuh; default when eligible)
// and the score pass + PDL-chained sampler pair (fp32 caches, page sizes not a multiple of 64,
// contexts > 64k, profiling, and the sequence-sharded phases).

constexpr int kTcMinHeads = 1024;  // AUTO runs the tcgen05 step kernel from here (and S <= 256)

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct WsLayout {
  int L = 64, Cmax = 0, Cmax256 = 0;
  size_t stash = 0, cstats = 0, tickets = 0, flags = 0, sync = 0, bern = 0, total = 0;
  size_t step_rec = 0, step_stash = 0, step_part = 0;  // step kernel's tagged regions
};

constexpr int kMaxSeqlen = 1 << 20;   // chunk-CDF tables are sized for <= 8192 chunks of <= 128 keys

int elem_bytes(int dtype) { return dtype == SANTA_F32 ? 4 : 2; }

santa_status validate_geometry(const santa_geometry* g) {
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

WsLayout layout(const santa_geometry* g, int S) {
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
  // step kernel: tagged chunk records, tagged fixed-point stash, tagged split partials (separate
  // from the two-kernel path's untagged regions so the paths can share one workspace)
  L.step_rec = off; off = align256(off + B * H * (size_t)L.Cmax * 16);
  L.step_stash = off; off = align256(off + B * H * (size_t)L.Cmax * 64 * 4);
  L.step_part = off; off = align256(off + B * H * (size_t)kStepMaxSplits * D * 8);
  L.total = off;
  return L;
}

santa_status check_ws(const santa_geometry* g, int S, void* ws, size_t ws_bytes, WsLayout* L) {
  *L = layout(g, S);
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255u)) return SANTA_ERR_WORKSPACE;
  if (ws_bytes < L->total) return SANTA_ERR_WORKSPACE;
  return SANTA_OK;
}

template <typename P>
P* at(void* ws, size_t off) { return reinterpret_cast<P*>(reinterpret_cast<char*>(ws) + off); }

KvLayout kv_layout(const santa_geometry* g) {
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

float scale_log2(const santa_geometry* g) {
  const float s = g->scale > 0.f ? g->scale : 1.0f / std::sqrt((float)g->head_dim);
  return s * kLog2e;
}

santa_status last_cuda() {
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
santa_status dispatch(int dtype, int D, int G, A&&... a) {
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
};

// ---- host-side caches: per device, safe under concurrent calls from several host threads ----
// (santa.h promises reentrancy: the only process-wide state is these caches of facts about the
// device and the kernels, each written idempotently.)
constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev;
}

int num_sms() {
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
std::mutex g_attr_mu;

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
bool fits_one_per_sm(Kern kern, int nthreads, size_t smem) {
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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
bool make_kmap(CUtensorMap* m, const void* K, uint64_t rows, int D, int dtype, int box_rows = 64) {
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
bool make_qmap(CUtensorMap* m, const void* q, uint64_t rows, int D, int dtype, int G) {
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

ScoreParams make_score_params(const DecodeArgs& a) {
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

bool stream_eligible(const santa_geometry* g) {
  return g->dtype != SANTA_F32 && (!g->page_table || g->page_size % kStageKeys == 0);
}

template <typename T, int D, int G>
struct RunScore {
  static santa_status run(const DecodeArgs& a) {
    ScoreParams p = make_score_params(a);
    if (a.events) cudaEventRecord(a.events[0], a.st);
    const bool stream = !a.g->page_table || a.g->page_size % kStageKeys == 0;
    if constexpr (sizeof(T) == 2) if (stream) {
      CUtensorMap tm;
      const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                            : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
      if (!make_kmap(&tm, a.K, rows, D, a.g->dtype)) return SANTA_ERR_CUDA;
      constexpr size_t kStageBytes = (D / 64) * 8192;
      constexpr int NW = kStreamWarps, SPW = kStreamSlots;
      const size_t smem = 1024 + (size_t)NW * G * p.L * 4 + (size_t)NW * SPW * (kStageBytes + 16);
      if (smem <= 220 * 1024) {  // else: per-warp score buffers too large (G * L big) -> fallback kernel
      if (ensure_smem(score_stream_kernel<T, D, G, NW, SPW>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
      const int total = a.g->batch * a.g->n_kv_heads * p.Cmax;
      const int grid = total < num_sms() ? total : num_sms();
      if (launch(score_stream_kernel<T, D, G, NW, SPW>, dim3(grid), dim3(32 * (NW + 1)), smem, a.st, false, tm, p) !=
          cudaSuccess)
        return SANTA_ERR_CUDA;
      return SANTA_OK;
      }
    }
    {
      dim3 grid(a.L.Cmax, a.g->n_kv_heads, a.g->batch);
      const size_t smem = (size_t)G * p.L * 4;
      if (ensure_smem(score_chunk_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
      if (launch(score_chunk_kernel<T, D, G>, grid, dim3(128), smem, a.st, false, p) != cudaSuccess)
        return SANTA_ERR_CUDA;
    }
    return SANTA_OK;
  }
};

SampleParams make_sample_params(const DecodeArgs& a) {
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
  p.trace = nullptr;
  p.cluster = 1;
  return p;
}

template <typename T, int D, int G>
struct RunSample {
  static santa_status run(const DecodeArgs& a) {
    SampleParams p = make_sample_params(a);
    // CTAs per head: a thread-block cluster of CS CTAs splits the S strata (more SMs on the
    // latency-bound search/gather), partials summed through DSMEM.  Aim at >= ~2 CTAs per SM.
    int CS = 1;
    const int heads = a.g->batch * a.g->n_heads;
    while (CS < 4 && heads * CS * 2 <= 2 * num_sms() && CS * 2 <= a.S) CS *= 2;
    p.cluster = CS;
    const size_t smem = sample_smem_bytes(p.Cmax, (a.S + CS - 1) / CS, D, kSampleThreads);
    if (ensure_smem(sample_gather_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    if (a.events) cudaEventRecord(a.events[1], a.st);
    const bool pdl = a.events == nullptr && a.stats_all == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.g->n_heads * CS, a.g->batch);
    cfg.blockDim = dim3(kSampleThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CS;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    if (cudaLaunchKernelEx(&cfg, sample_gather_kernel<T, D, G>, p) != cudaSuccess) return SANTA_ERR_CUDA;
    if (a.events) cudaEventRecord(a.events[2], a.st);
    return SANTA_OK;
  }
};

// S^2ANTA-prop budgets + counts + gather (prop_kernels.cuh), PDL-chained to the score pass; the
// same cluster split of the S samples as RunSample.
template <typename T, int D, int G>
struct RunProp {
  static santa_status run(const DecodeArgs& a) {
    SampleParams p = make_sample_params(a);
    int CS = 1;
    const int heads = a.g->batch * a.g->n_heads;
    while (CS < 4 && heads * CS * 2 <= 2 * num_sms() && CS * 2 <= a.S) CS *= 2;
    p.cluster = CS;
    const size_t smem = prop_smem_bytes(p.Cmax, (a.S + CS - 1) / CS, D, kSampleThreads);
    if (smem > 227 * 1024) return SANTA_ERR_UNSUPPORTED;
    if (ensure_smem(prop_gather_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.g->n_heads * CS, a.g->batch);
    cfg.blockDim = dim3(kSampleThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, prop_gather_kernel<T, D, G>, p) != cudaSuccess) return SANTA_ERR_CUDA;
    return SANTA_OK;
  }
};

// S^2ANTA-flash per-tile draws + merge-weighted gather (flash_kernels.cuh), PDL-chained to the
// score pass.  cpt = chunks per flash tile, mmax = idx row length (santa_flash_max_samples).
template <typename T, int D, int G>
struct RunFlash {
  static santa_status run(const DecodeArgs& a, int cpt, int mmax) {
    SampleParams p = make_sample_params(a);
    int CS = 1;
    const int heads = a.g->batch * a.g->n_heads;
    // up to 4 CTAs per head within one wave (8-CTA clusters measured slower: 132 registers x 256
    // threads fit one CTA per SM, so 256 CTAs ran in two waves)
    while (CS < 4 && heads * CS * 2 <= 2 * num_sms() && CS * 2 <= mmax) CS *= 2;
    p.cluster = CS;
    const size_t smem = flash_smem_bytes(p.Cmax, cpt, (mmax + CS - 1) / CS, D, kSampleThreads);
    if (smem > 227 * 1024) return SANTA_ERR_UNSUPPORTED;
    if (ensure_smem(flash_gather_kernel<T, D, G>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.g->n_heads * CS, a.g->batch);
    cfg.blockDim = dim3(kSampleThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, flash_gather_kernel<T, D, G>, p, cpt, mmax) != cudaSuccess) return SANTA_ERR_CUDA;
    return SANTA_OK;
  }
};

// idx row length of the flash path: max over sequence lengths <= max_seqlen of S_tile * T
// (-1: tile_len is not a positive multiple of the chunk length, or more than 64 chunks).
int flash_max_samples(const santa_geometry* g, int S, int tile_len, int* cpt_out) {
  const int L = layout(g, 1).L;
  if (tile_len < L || tile_len % L != 0 || tile_len / L > 64 || S < 1) return -1;
  const int cpt = tile_len / L;
  const int Tmax = (g->max_seqlen + tile_len - 1) / tile_len;
  int mm = 0;
  for (int T = 1; T <= Tmax; ++T) {
    const int m = flash_tile_budget(T, S) * T;
    if (m > mm) mm = m;
  }
  if (cpt_out) *cpt_out = cpt;
  return mm;
}

// The whole step in one pipelined cooperative launch (step_kernel.cuh).  Returns
// SANTA_ERR_UNSUPPORTED (nothing launched) when the configuration does not qualify, in which
// case the caller runs the two-kernel path.
// A cooperative launch the device cannot co-schedule (e.g. SMs held by another context) is
// "unsupported here", not a failure: AUTO then runs the two-kernel path.
santa_status coop_status(cudaError_t e) {
  if (e == cudaSuccess) return SANTA_OK;
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();  // clear the sticky-free launch error
    return SANTA_ERR_UNSUPPORTED;
  }
  return SANTA_ERR_CUDA;
}

StepSync make_step_sync(const DecodeArgs& a) {
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

template <typename T, int D, int G>
struct RunStep {
  // the tensor-core variant (santa_step_tc_kernel): 128-key tiles, pages of a multiple of 128
  static santa_status run_tc(const DecodeArgs& a, const ScoreParams& sp, const SampleParams& pp, int CS, int grid) {
    if constexpr (sizeof(T) != 2) {
      return SANTA_ERR_UNSUPPORTED;
    } else {
      constexpr int NSW = kStepSamplers, NT = 32 * kTcWarps;
      if (a.g->page_table && a.g->page_size % kTcTileKeys != 0) return SANTA_ERR_UNSUPPORTED;
      const size_t smem = step_tc_score_smem_bytes(D, G) + step_sample_smem_bytes(pp.Cmax, (a.S + CS - 1) / CS, D);
      if (smem > 226 * 1024) return SANTA_ERR_UNSUPPORTED;
      auto kern = santa_step_tc_kernel<T, D, G, NSW>;
      if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
      if (!fits_one_per_sm(kern, NT, smem)) return SANTA_ERR_UNSUPPORTED;
      CUtensorMap tk, tq;
      const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                            : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
      if (!make_kmap(&tk, a.K, rows, D, a.g->dtype, 64)) return SANTA_ERR_UNSUPPORTED;
      if (!make_qmap(&tq, a.q, (uint64_t)a.g->batch * a.g->n_heads, D, a.g->dtype, G)) return SANTA_ERR_UNSUPPORTED;
      StepSync sy = make_step_sync(a);
      SampleParams pq = pp;
      pq.cluster = CS;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = a.st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return coop_status(cudaLaunchKernelEx(&cfg, kern, tk, tq, sp, pq, sy));
    }
  }

  static santa_status run(const DecodeArgs& a) {
    if constexpr (sizeof(T) != 2) {
      return SANTA_ERR_UNSUPPORTED;
    } else {
      if (!stream_eligible(a.g) || a.L.L != kStepStageKeys) return SANTA_ERR_UNSUPPORTED;
      // the sampler group's chunk-CDF registers hold <= kStepMaxChunks chunks (65,536 tokens)
      if (a.L.Cmax > kStepMaxChunks) return SANTA_ERR_UNSUPPORTED;
      constexpr int NW = kStepConsumers, SPW = kStepSlots, NSW = kStepSamplers, NT = 32 * (NW + 1 + NSW);
      ScoreParams sp = make_score_params(a);
      SampleParams pp = make_sample_params(a);
      // splits per head: aim at one sampler round (<= 64 strata) per item, so the exposed tail (the
      // last unit's items) is one gather round, but keep the total at <= 4 items per CTA: every item
      // repeats the chunk-CDF combine, and at large batch the sampler work must stay hidden under
      // the stream (config 3, S = 512: 8192 items -> 661 us vs 1024 items -> see DESIGN.md sec. 5)
      const int grid = num_sms(), heads = a.g->batch * a.g->n_heads;
      int CS = 1;
      while (CS * 2 <= kStepMaxSplits && CS * 64 < a.S && heads * CS * 2 <= 4 * grid) CS *= 2;
      pp.cluster = CS;
      if (a.tensor_core) return run_tc(a, sp, pp, CS, grid);
      const size_t smem = step_score_smem_bytes(D, G, NW, SPW) + step_sample_smem_bytes(pp.Cmax, (a.S + CS - 1) / CS, D);
      if (smem > 226 * 1024) return SANTA_ERR_UNSUPPORTED;  // 227 KiB per CTA minus static smem
      auto kern = santa_step_kernel<T, D, G, NW, SPW, NSW>;
      if (ensure_smem(kern, smem) != cudaSuccess) return SANTA_ERR_CUDA;
      if (!fits_one_per_sm(kern, NT, smem)) return SANTA_ERR_UNSUPPORTED;
      CUtensorMap tm;
      const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                            : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
      if (!make_kmap(&tm, a.K, rows, D, a.g->dtype, kStepStageKeys)) return SANTA_ERR_UNSUPPORTED;
      StepSync sy = make_step_sync(a);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = a.st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return coop_status(cudaLaunchKernelEx(&cfg, kern, tm, sp, pp, sy));
    }
  }
};

template <typename T, int D, int G>
struct RunDense {
  static santa_status run(const DecodeArgs& a) {
    DenseParams p;
    p.q = a.q;
    p.K = a.K;
    p.V = a.V;
    p.kv = kv_layout(a.g);
    p.seqlens = a.seqlens;
    p.B = a.g->batch;
    p.H = a.g->n_heads;
    p.Hkv = a.g->n_kv_heads;
    p.scale_log2 = scale_log2(a.g);
    p.cstats = at<float2>(a.ws, a.L.cstats);
    p.opart = at<float>(a.ws, a.L.stash);
    p.Cmax = a.L.Cmax256;
    p.out = a.out;
    p.flags = at<uint32_t>(a.ws, a.L.flags);
    bool done = false;
    if constexpr (sizeof(T) == 2) {
      if (stream_eligible(a.g)) {  // tensor-core streaming flash-decoding kernel
        constexpr int NW = kDenseWarps, SPW = kDenseSlots;
        constexpr size_t kStageBytes = 2 * (D / 64) * kDenseStageKeys * 128;
        const size_t smem = 1024 + (size_t)NW * SPW * (kStageBytes + 16) + (size_t)NW * 8 * kPRow * 2;
        if (ensure_smem(dense_stream_kernel<T, D, G, NW, SPW>, smem) != cudaSuccess) return SANTA_ERR_CUDA;
        CUtensorMap tk, tv;
        const uint64_t rows = a.g->page_table ? (uint64_t)0x7fffffff
                                              : (uint64_t)a.g->batch * a.g->n_kv_heads * a.g->max_seqlen;
        if (!make_kmap(&tk, a.K, rows, D, a.g->dtype, kDenseStageKeys) ||
            !make_kmap(&tv, a.V, rows, D, a.g->dtype, kDenseStageKeys))
          return SANTA_ERR_CUDA;
        DenseStreamParams dp;
        dp.q = a.q;
        dp.kv = p.kv;
        dp.seqlens = a.seqlens;
        dp.B = p.B;
        dp.H = p.H;
        dp.Hkv = p.Hkv;
        dp.scale_log2 = p.scale_log2;
        dp.cstats = p.cstats;
        dp.opart = p.opart;
        dp.Cmax = p.Cmax;
        dp.flags = p.flags;
        const int total = a.g->batch * a.g->n_kv_heads * p.Cmax;
        const int grid = total < num_sms() ? total : num_sms();
        if (launch(dense_stream_kernel<T, D, G, NW, SPW>, dim3(grid), dim3(32 * (NW + 1)), smem, a.st, false, tk, tv,
                   dp) != cudaSuccess)
          return SANTA_ERR_CUDA;
        done = true;
      }
    }
    if (!done) {
      dim3 grid(a.L.Cmax256, a.g->n_kv_heads, a.g->batch);
      if (launch(dense_partial_kernel<T, D, G>, grid, dim3(kScoreThreads), 0, a.st, false, p) != cudaSuccess)
        return SANTA_ERR_CUDA;
    }
    if (launch(dense_combine_kernel<T, D>, dim3(a.g->n_heads, a.g->batch), dim3(256), 0, a.st, true, p) !=
        cudaSuccess)
      return SANTA_ERR_CUDA;
    return SANTA_OK;
  }
};

// local shard combine: (m_r, L_r) per (b, h) from the chunk stats, fp64
__global__ void shard_combine_kernel(const float2* __restrict__ cstats, const int32_t* __restrict__ seqlens,
                                     int H, int Cmax, int L, double* __restrict__ stats_out) {
  pdl_wait_primary();
  const int h = blockIdx.x, b = blockIdx.y;
  const int seqlen = __ldg(seqlens + b);
  const int nC = seqlen > 0 ? (seqlen + L - 1) / L : 0;
  const float2* cs = cstats + ((size_t)b * H + h) * Cmax;
  __shared__ double red[32];
  float m = -INFINITY;
  for (int c = threadIdx.x; c < nC; c += blockDim.x) m = fmaxf(m, __ldcg(&cs[c].x));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  float mm = -INFINITY;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mm = fmaxf(mm, (float)red[w]);
  __syncthreads();
  double s = 0.0;
  for (int c = threadIdx.x; c < nC; c += blockDim.x) {
    const float2 st = __ldcg(&cs[c]);
    if (st.y > 0.f) s += exp2((double)st.x - (double)mm) * (double)st.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];  // fixed order
    stats_out[((size_t)b * H + h) * 2] = nC ? (double)mm : -INFINITY;
    stats_out[((size_t)b * H + h) * 2 + 1] = nC ? t : 0.0;
  }
}

__global__ void append_kv_kernel(void* K, void* V, const void* kn, const void* vn, KvLayout kv,
                                 const int32_t* seqlens, int D, int eb) {
  const int kvh = blockIdx.x, b = blockIdx.y;
  const int t = __ldg(seqlens + b) - 1;
  if (t < 0) return;
  const int64_t dst = kv.row(b, kvh, t, D) * eb;
  const int64_t src = ((int64_t)b * kv.n_kv_heads + kvh) * D * eb;
  for (int i = threadIdx.x; i < D * eb; i += blockDim.x) {
    reinterpret_cast<char*>(K)[dst + i] = reinterpret_cast<const char*>(kn)[src + i];
    reinterpret_cast<char*>(V)[dst + i] = reinterpret_cast<const char*>(vn)[src + i];
  }
}

// Zero-copy staging for the packed host API: one CTA per (b, kv head) reads its G query rows and
// its new K/V rows straight from the PINNED host buffer (a device-addressable alias under UVA) with
// 16-B loads, writes the q rows to the device staging buffer and the K/V rows into the cache slot
// seqlens[b] - 1 -- the H2D copy and the append in one launch.
__global__ void stage_append_kernel(const uint4* __restrict__ qkv_h, uint4* __restrict__ q_dev, void* K, void* V,
                                    KvLayout kv, const int32_t* seqlens, int D, int eb, int G, int H) {
  const int kvh = blockIdx.x, b = blockIdx.y, Hkv = kv.n_kv_heads;
  const int row16 = D * eb / 16;                                 // 16-B words per row
  const size_t q16 = (size_t)gridDim.y * H * row16, k16 = (size_t)gridDim.y * Hkv * row16;
  const size_t qsrc = ((size_t)b * H + (size_t)kvh * G) * row16;
  for (int i = threadIdx.x; i < G * row16; i += blockDim.x) q_dev[qsrc + i] = qkv_h[qsrc + i];
  const int t = __ldg(seqlens + b) - 1;
  if (t < 0) return;
  const int64_t dst16 = kv.row(b, kvh, t, D) * eb / 16;
  const size_t ksrc = q16 + ((size_t)b * Hkv + kvh) * row16;
  for (int i = threadIdx.x; i < row16; i += blockDim.x) {
    reinterpret_cast<uint4*>(K)[dst16 + i] = qkv_h[ksrc + i];
    reinterpret_cast<uint4*>(V)[dst16 + i] = qkv_h[ksrc + k16 + i];
  }
}

// The device-addressable alias of a page-locked host pointer (cudaHostAlloc / cudaHostRegister,
// e.g. torch pin_memory), or NULL for pageable memory.  Queried per call (no cache: a freed pinned
// buffer's address can come back as pageable memory).
const void* pinned_alias(const void* hp) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, hp) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

__global__ void philox_test_kernel(uint64_t seed, uint64_t offset, uint32_t tag, uint32_t h, uint32_t b, int n,
                                   double* out, uint4 ctr, uint2 key, uint32_t* raw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  PhiloxStream ps(seed, offset, tag, h, b);
  if (i < n) out[i] = ps.uniform((uint32_t)i);
  if (raw && i == 0) {
    const Philox4 o = philox4x32_10(ctr.x, ctr.y, ctr.z, ctr.w, key.x, key.y);
    raw[0] = o.x[0]; raw[1] = o.x[1]; raw[2] = o.x[2]; raw[3] = o.x[3];
  }
}

santa_status validate_decode_ptrs(const void* q, const void* K, const void* V, const int32_t* seqlens,
                                  const void* out) {
  if (!q || !K || !V || !seqlens || !out) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(K) || !aligned16(V) || !aligned16(out)) return SANTA_ERR_ALIGNMENT;
  if (reinterpret_cast<uintptr_t>(seqlens) & 3u) return SANTA_ERR_ALIGNMENT;
  return SANTA_OK;
}

template <typename T, int D, int G>
struct RunBern {
  // mode 0: standalone scores (scores != NULL, no stash); mode 1: fused into the decode step
  static santa_status run(const DecodeArgs& a, const void* Kt, int nB, int stratified, int mean_group,
                          float* scores, uint8_t* mask, bool for_decode) {
    BernParams p = {};
    p.q = a.q;
    p.Kt = Kt;
    p.seqlens = a.seqlens;
    p.B = a.g->batch;
    p.H = a.g->n_heads;
    p.Hkv = a.g->n_kv_heads;
    p.nB = nB;
    p.stratified = stratified;
    p.mean_group = mean_group;
    p.seed = a.seed;
    p.offset = a.offset;
    p.batch_offset = a.g->batch_offset;
    p.head_offset = a.g->head_offset;
    p.scale = a.g->scale > 0.f ? a.g->scale : 1.0f / std::sqrt((float)D);
    char* bern = at<char>(a.ws, a.L.bern);
    const size_t units = (size_t)a.g->batch * a.g->n_kv_heads;
    p.w = reinterpret_cast<float*>(bern);
    p.sel = reinterpret_cast<int*>(bern + units * G * D * 4);
    p.sel_n = reinterpret_cast<int*>(bern + units * G * D * 4 + units * D * 4);
    p.feature_mask = mask;
    p.page_table = a.g->page_table;
    p.page_size = a.g->page_size;
    p.max_pages = a.g->max_pages_per_seq;
    p.scores = scores;
    p.score_stride = a.g->max_seqlen;
    p.stash = for_decode ? at<float>(a.ws, a.L.stash) : nullptr;
    p.cstats = at<float2>(a.ws, a.L.cstats);
    // decode: 64-key stats/stash in the standard layout when L = 64 (the sampler's fast ballot
    // search), else per 256-key chunk
    p.sub64 = (for_decode && a.L.L == 64) ? 1 : 0;
    p.Cmax = p.sub64 ? a.L.Cmax : a.L.Cmax256;
    p.stash_stride = p.sub64 ? a.L.Cmax * 64 : a.L.Cmax256 * kDenseChunk;
    p.tickets = at<uint32_t>(a.ws, a.L.tickets);
    p.flags = at<uint32_t>(a.ws, a.L.flags);
    if (launch(bern_weights_kernel<T, D, G>, dim3(a.g->n_kv_heads, a.g->batch), dim3(D), 0, a.st, false, p) !=
        cudaSuccess)
      return SANTA_ERR_CUDA;
    if (launch(bern_chunk_kernel<T, D, G>, dim3(a.L.Cmax256, a.g->n_kv_heads, a.g->batch), dim3(kScoreThreads), 0,
               a.st, true, p) != cudaSuccess)
      return SANTA_ERR_CUDA;
    return SANTA_OK;
  }
};

santa_status validate_bern(const santa_geometry* g, const void* q, const void* Kt, const int32_t* seqlens,
                           int32_t nB) {
  if (!q || !Kt || !seqlens) return SANTA_ERR_INVALID_ARG;
  if (nB < 1) return SANTA_ERR_EMPTY_BUDGET;
  if (nB > 4096) return SANTA_ERR_UNSUPPORTED;
  if (!aligned16(q) || !aligned16(Kt)) return SANTA_ERR_ALIGNMENT;
  if (!g->page_table && (g->max_seqlen % 8) != 0) return SANTA_ERR_SHAPE;  // 16-B aligned feature rows
  return SANTA_OK;
}

int auto_path(const santa_geometry* g, int S) {
  const bool step_ok = g->dtype != SANTA_F32 && g->max_seqlen <= 65536;
  const bool tc_pages = !g->page_table || g->page_size % kTcTileKeys == 0;
  if (step_ok && (int64_t)g->batch * g->n_heads >= kTcMinHeads) {
    // batch 32 (tools/path_sweep.py, profiles/r01_v10_path_sweep_*.json): S <= 256 the tcgen05 step
    // kernel (367 / 383-393 us at S = 64 / 256), S = 512 the mma.sync step kernel (419 vs 437 us for
    // the two-kernel path, 458 for tcgen05)
    if (S <= 256 && tc_pages) return SANTA_PATH_STEP_TC;
    if (S > 256 && S <= 512) return SANTA_PATH_STEP_KERNEL;
  }
  return SANTA_PATH_TWO_KERNEL;
}

// Every check santa_decode_attention makes, with no side effect: fills *a on success.  The host-buffer
// entry points call it BEFORE their first copy or launch (santa.h: on any error nothing is launched).
santa_status prepare_decode(const santa_geometry* g, const void* q, const void* K, const void* V,
                            const int32_t* seqlens, int32_t S, int32_t mode, uint64_t seed, uint64_t offset,
                            void* out, int32_t* idx_out, void* ws, size_t ws_bytes, void* const* events,
                            void* stream, int path, DecodeArgs* a) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (path < SANTA_PATH_AUTO || path > SANTA_PATH_STEP_TC) return SANTA_ERR_INVALID_ARG;
  if (S < 1) return SANTA_ERR_EMPTY_BUDGET;
  if (S > kMaxBudget) return SANTA_ERR_UNSUPPORTED;
  if (mode < SANTA_IID || mode > SANTA_SYSTEMATIC) return SANTA_ERR_INVALID_ARG;
  if ((s = validate_decode_ptrs(q, K, V, seqlens, out)) != SANTA_OK) return s;
  if (idx_out && (reinterpret_cast<uintptr_t>(idx_out) & 3u)) return SANTA_ERR_ALIGNMENT;
  *a = DecodeArgs{};
  if ((s = check_ws(g, S, ws, ws_bytes, &a->L)) != SANTA_OK) return s;
  a->g = g; a->q = q; a->K = K; a->V = V; a->seqlens = seqlens; a->S = S; a->mode = mode;
  a->seed = seed; a->offset = offset; a->out = out; a->idx_out = idx_out; a->ws = ws;
  a->st = reinterpret_cast<cudaStream_t>(stream);
  a->events = reinterpret_cast<cudaEvent_t const*>(events);
  return SANTA_OK;
}

// Launch a prepared decode step on `path` (AUTO resolved here).
santa_status run_decode(DecodeArgs& a, int path) {
  const santa_geometry* g = a.g;
  const bool auto_requested = path == SANTA_PATH_AUTO;
  const int G = g->n_heads / g->n_kv_heads;
  santa_status s;
  // AUTO (measured, tools/path_sweep.py -> profiles/r01_v6_path_sweep.json): the tcgen05 step kernel
  // from 1024 query heads per call with S <= 256 (batch 32: 391 vs 403 us); below that, the score
  // pass + PDL-chained sampler (batch 1: 25.0 vs 26.8 us for the mma.sync step kernel) -- the
  // sampler kernel then has every SM for the final sampling chain
  if (path == SANTA_PATH_AUTO) path = auto_path(g, a.S);
  if (!a.events && path != SANTA_PATH_TWO_KERNEL) {
    a.tensor_core = path == SANTA_PATH_STEP_TC;
    s = dispatch<RunStep>(g->dtype, g->head_dim, G, a);
    if (s == SANTA_ERR_UNSUPPORTED && a.tensor_core && auto_requested) {
      a.tensor_core = false;  // e.g. pages not a multiple of 128 tokens
      s = dispatch<RunStep>(g->dtype, g->head_dim, G, a);
    }
    if (s == SANTA_OK) return last_cuda();
    if (s != SANTA_ERR_UNSUPPORTED || !auto_requested) return s;
  }
  if ((s = dispatch<RunScore>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  if ((s = dispatch<RunSample>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  return last_cuda();
}

santa_status decode_common(const santa_geometry* g, const void* q, const void* K, const void* V,
                           const int32_t* seqlens, int32_t S, int32_t mode, uint64_t seed, uint64_t offset,
                           void* out, int32_t* idx_out, void* ws, size_t ws_bytes, void* const* events,
                           void* stream, int path = SANTA_PATH_AUTO) {
  DecodeArgs a;
  const santa_status s =
      prepare_decode(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, events, stream, path, &a);
  if (s != SANTA_OK) return s;
  return run_decode(a, path);
}

}  // namespace

extern "C" {

const char* santa_status_string(santa_status s) {
  switch (s) {
    case SANTA_OK: return "SANTA_OK";
    case SANTA_ERR_INVALID_ARG: return "SANTA_ERR_INVALID_ARG";
    case SANTA_ERR_SHAPE: return "SANTA_ERR_SHAPE";
    case SANTA_ERR_EMPTY_BUDGET: return "SANTA_ERR_EMPTY_BUDGET";
    case SANTA_ERR_EMPTY_DISTRIBUTION: return "SANTA_ERR_EMPTY_DISTRIBUTION";
    case SANTA_ERR_UNSUPPORTED: return "SANTA_ERR_UNSUPPORTED";
    case SANTA_ERR_WORKSPACE: return "SANTA_ERR_WORKSPACE";
    case SANTA_ERR_ALIGNMENT: return "SANTA_ERR_ALIGNMENT";
    case SANTA_ERR_CUDA: return "SANTA_ERR_CUDA";
  }
  return "SANTA_ERR_UNKNOWN";
}

const char* santa_version(void) {
  return "libsanta 0.3 sm_100a (santa_step_kernel: single-launch persistent step, tagged-word publication; santa_step_tc_kernel: tcgen05 score stage, TMEM accumulators; score_stream: TMA 128B-swizzle ring + mma.sync, interleaved; sample_gather: thread-block clusters; prop/flash: S^2ANTA-prop and -flash tile estimators; dense: TMA flash-decoding; bernoulli)";
}

int32_t santa_auto_path(const santa_geometry* g, int32_t S) {
  if (validate_geometry(g) != SANTA_OK || S < 1) return -1;
  return auto_path(g, S);
}

size_t santa_workspace_bytes(const santa_geometry* g, int32_t S) {
  if (validate_geometry(g) != SANTA_OK || S < 1) return 0;
  return layout(g, S).total;
}

santa_status santa_decode_attention(const santa_geometry* g, const void* q, const void* K, const void* V,
                                    const int32_t* seqlens, int32_t S, int32_t mode, uint64_t seed,
                                    uint64_t offset, void* out, int32_t* idx_out, void* ws, size_t ws_bytes,
                                    void* stream) {
  return decode_common(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, nullptr, stream);
}

santa_status santa_decode_attention_path(const santa_geometry* g, const void* q, const void* K, const void* V,
                                         const int32_t* seqlens, int32_t S, int32_t mode, uint64_t seed,
                                         uint64_t offset, void* out, int32_t* idx_out, void* ws, size_t ws_bytes,
                                         int32_t path, void* stream) {
  return decode_common(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, nullptr, stream,
                       path);
}

santa_status santa_decode_attention_profiled(const santa_geometry* g, const void* q, const void* K,
                                             const void* V, const int32_t* seqlens, int32_t S, int32_t mode,
                                             uint64_t seed, uint64_t offset, void* out, int32_t* idx_out,
                                             void* ws, size_t ws_bytes, void* const* events, void* stream) {
  if (!events || !events[0] || !events[1] || !events[2]) return SANTA_ERR_INVALID_ARG;
  return decode_common(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, events, stream);
}

santa_status santa_score_phase(const santa_geometry* g, const void* q, const void* K, const int32_t* seqlens,
                               void* ws, size_t ws_bytes, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (!q || !K || !seqlens) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(K)) return SANTA_ERR_ALIGNMENT;
  DecodeArgs a = {};
  if ((s = check_ws(g, 1, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.q = q; a.K = K; a.seqlens = seqlens; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunScore>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  return last_cuda();
}

santa_status santa_sample_phase(const santa_geometry* g, const void* V, const int32_t* seqlens, int32_t S,
                                int32_t mode, uint64_t seed, uint64_t offset, void* out, int32_t* idx_out, void* ws,
                                size_t ws_bytes, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (S < 1) return SANTA_ERR_EMPTY_BUDGET;
  if (S > kMaxBudget) return SANTA_ERR_UNSUPPORTED;
  if (mode < SANTA_IID || mode > SANTA_SYSTEMATIC) return SANTA_ERR_INVALID_ARG;
  if (!V || !seqlens || !out) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(V) || !aligned16(out)) return SANTA_ERR_ALIGNMENT;
  DecodeArgs a = {};
  if ((s = check_ws(g, S, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.V = V; a.seqlens = seqlens; a.S = S; a.mode = mode; a.seed = seed; a.offset = offset; a.out = out;
  a.idx_out = idx_out; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunSample>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  return last_cuda();
}

santa_status santa_decode_attention_prop(const santa_geometry* g, const void* q, const void* K, const void* V,
                                         const int32_t* seqlens, int32_t S, uint64_t seed, uint64_t offset,
                                         void* out, int32_t* idx_out, void* ws, size_t ws_bytes, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (S < 1) return SANTA_ERR_EMPTY_BUDGET;
  if (S > kMaxBudget) return SANTA_ERR_UNSUPPORTED;
  if ((s = validate_decode_ptrs(q, K, V, seqlens, out)) != SANTA_OK) return s;
  if (idx_out && (reinterpret_cast<uintptr_t>(idx_out) & 3u)) return SANTA_ERR_ALIGNMENT;
  DecodeArgs a = {};
  if ((s = check_ws(g, S, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.q = q; a.K = K; a.V = V; a.seqlens = seqlens; a.S = S; a.mode = SANTA_SYSTEMATIC;
  a.seed = seed; a.offset = offset; a.out = out; a.idx_out = idx_out; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunScore>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  if ((s = dispatch<RunProp>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  return last_cuda();
}

int32_t santa_prop_tile_len(const santa_geometry* g) {
  if (validate_geometry(g) != SANTA_OK) return -1;
  return layout(g, 1).L;
}

santa_status santa_decode_attention_flash(const santa_geometry* g, const void* q, const void* K, const void* V,
                                          const int32_t* seqlens, int32_t S, int32_t tile_len, uint64_t seed,
                                          uint64_t offset, void* out, int32_t* idx_out, void* ws, size_t ws_bytes,
                                          void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (S < 1) return SANTA_ERR_EMPTY_BUDGET;
  if (S > kMaxBudget) return SANTA_ERR_UNSUPPORTED;
  int cpt = 0;
  const int mmax = flash_max_samples(g, S, tile_len, &cpt);
  if (mmax < 0) return SANTA_ERR_INVALID_ARG;
  if (mmax > 16384) return SANTA_ERR_UNSUPPORTED;
  if ((s = validate_decode_ptrs(q, K, V, seqlens, out)) != SANTA_OK) return s;
  if (idx_out && (reinterpret_cast<uintptr_t>(idx_out) & 3u)) return SANTA_ERR_ALIGNMENT;
  DecodeArgs a = {};
  if ((s = check_ws(g, S, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.q = q; a.K = K; a.V = V; a.seqlens = seqlens; a.S = S; a.mode = SANTA_SYSTEMATIC;
  a.seed = seed; a.offset = offset; a.out = out; a.idx_out = idx_out; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunScore>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  if ((s = dispatch<RunFlash>(g->dtype, g->head_dim, G, a, cpt, mmax)) != SANTA_OK) return s;
  return last_cuda();
}

int32_t santa_flash_max_samples(const santa_geometry* g, int32_t S, int32_t tile_len) {
  if (validate_geometry(g) != SANTA_OK) return -1;
  return flash_max_samples(g, S, tile_len, nullptr);
}

santa_status santa_dense_reference(const santa_geometry* g, const void* q, const void* K, const void* V,
                                   const int32_t* seqlens, void* out, void* ws, size_t ws_bytes, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if ((s = validate_decode_ptrs(q, K, V, seqlens, out)) != SANTA_OK) return s;
  DecodeArgs a = {};
  if ((s = check_ws(g, 1, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.q = q; a.K = K; a.V = V; a.seqlens = seqlens; a.out = out; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunDense>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  return last_cuda();
}

santa_status santa_bernoulli_scores(const santa_geometry* g, const void* q, const void* Kt, const int32_t* seqlens,
                                    int32_t nB, int32_t stratified, int32_t mean_group, uint64_t seed,
                                    uint64_t offset, float* scores, uint8_t* feature_mask, void* ws,
                                    size_t ws_bytes, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if ((s = validate_bern(g, q, Kt, seqlens, nB)) != SANTA_OK) return s;
  if (!scores) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(scores)) return SANTA_ERR_ALIGNMENT;
  DecodeArgs a = {};
  if ((s = check_ws(g, 1, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.q = q; a.seqlens = seqlens; a.seed = seed; a.offset = offset; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunBern>(g->dtype, g->head_dim, G, a, Kt, (int)nB, (int)stratified, (int)mean_group, scores,
                             feature_mask, false)) != SANTA_OK)
    return s;
  return last_cuda();
}

santa_status santa_decode_attention_bernoulli(const santa_geometry* g, const void* q, const void* Kt, const void* V,
                                              const int32_t* seqlens, int32_t nB, int32_t stratified,
                                              int32_t mean_group, int32_t S, int32_t mode, uint64_t seed,
                                              uint64_t offset, void* out, int32_t* idx_out, void* ws,
                                              size_t ws_bytes, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if ((s = validate_bern(g, q, Kt, seqlens, nB)) != SANTA_OK) return s;
  if (S < 1) return SANTA_ERR_EMPTY_BUDGET;
  if (S > kMaxBudget) return SANTA_ERR_UNSUPPORTED;
  if (mode < SANTA_IID || mode > SANTA_SYSTEMATIC) return SANTA_ERR_INVALID_ARG;
  if ((s = validate_decode_ptrs(q, Kt, V, seqlens, out)) != SANTA_OK) return s;
  DecodeArgs a = {};
  if ((s = check_ws(g, S, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.q = q; a.V = V; a.seqlens = seqlens; a.S = S; a.mode = mode; a.seed = seed; a.offset = offset;
  a.out = out; a.idx_out = idx_out; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunBern>(g->dtype, g->head_dim, G, a, Kt, (int)nB, (int)stratified, (int)mean_group,
                             (float*)nullptr, (uint8_t*)nullptr, true)) != SANTA_OK)
    return s;
  if (a.L.L != 64) {  // stats per 256-key chunk (contexts > 512k)
    a.Lc = kDenseChunk;
    a.Cc = a.L.Cmax256;
  }
  if ((s = dispatch<RunSample>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  return last_cuda();
}

santa_status santa_seqshard_stats(const santa_geometry* g, const void* q, const void* K_shard,
                                  const int32_t* shard_seqlens, double* stats_out, void* ws, size_t ws_bytes,
                                  void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (!q || !K_shard || !shard_seqlens || !stats_out) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(K_shard) || !aligned16(stats_out)) return SANTA_ERR_ALIGNMENT;
  DecodeArgs a = {};
  if ((s = check_ws(g, 1, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.q = q; a.K = K_shard; a.seqlens = shard_seqlens; a.ws = ws;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunScore>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  if (launch(shard_combine_kernel, dim3(g->n_heads, g->batch), dim3(128), 0, a.st, true,
             (const float2*)at<float2>(ws, a.L.cstats), shard_seqlens, g->n_heads, a.L.Cmax, a.L.L, stats_out) !=
      cudaSuccess)
    return SANTA_ERR_CUDA;
  return last_cuda();
}

santa_status santa_seqshard_sample_gather(const santa_geometry* g, const double* stats_all, int32_t rank,
                                          int32_t world, const int32_t* token_offset, const void* V_shard,
                                          const int32_t* shard_seqlens, int32_t S, int32_t mode, uint64_t seed,
                                          uint64_t offset, float* partial_out, int32_t* idx_out, void* ws,
                                          size_t ws_bytes, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (S < 1) return SANTA_ERR_EMPTY_BUDGET;
  if (S > kMaxBudget) return SANTA_ERR_UNSUPPORTED;
  if (mode < SANTA_IID || mode > SANTA_SYSTEMATIC) return SANTA_ERR_INVALID_ARG;
  if (!stats_all || !V_shard || !shard_seqlens || !partial_out || !token_offset) return SANTA_ERR_INVALID_ARG;
  if (world < 1 || rank < 0 || rank >= world) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(V_shard) || !aligned16(partial_out)) return SANTA_ERR_ALIGNMENT;
  DecodeArgs a = {};
  // phase 2 must see the same chunk layout as phase 1 (which sized it with S = 1)
  if ((s = check_ws(g, S, ws, ws_bytes, &a.L)) != SANTA_OK) return s;
  a.g = g; a.V = V_shard; a.seqlens = shard_seqlens; a.S = S; a.mode = mode; a.seed = seed;
  a.offset = offset; a.out = partial_out; a.out_f32 = partial_out; a.idx_out = idx_out; a.ws = ws;
  a.stats_all = stats_all; a.rank = rank; a.world = world; a.token_offset = token_offset;
  a.st = reinterpret_cast<cudaStream_t>(stream);
  const int G = g->n_heads / g->n_kv_heads;
  if ((s = dispatch<RunSample>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
  return last_cuda();
}

santa_status santa_decode_step_host(const santa_geometry* g, const void* q_host, const void* k_new_host,
                                    const void* v_new_host, void* q_dev, void* k_new_dev, void* v_new_dev,
                                    void* K, void* V, const int32_t* seqlens, int32_t S, int32_t mode,
                                    uint64_t seed, uint64_t offset, void* out_dev, void* out_host, void* ws,
                                    size_t ws_bytes, void* stream) {
  if (!q_host || !k_new_host || !v_new_host || !q_dev || !k_new_dev || !v_new_dev || !out_host)
    return SANTA_ERR_INVALID_ARG;
  // the whole decode validation runs before the first copy (nothing is touched on error)
  DecodeArgs a;
  santa_status s = prepare_decode(g, q_dev, K, V, seqlens, S, mode, seed, offset, out_dev, nullptr, ws, ws_bytes,
                                  nullptr, stream, SANTA_PATH_AUTO, &a);
  if (s != SANTA_OK) return s;
  cudaStream_t st = a.st;
  const size_t eb = elem_bytes(g->dtype), D = g->head_dim;
  const size_t qb = (size_t)g->batch * g->n_heads * D * eb, kb = (size_t)g->batch * g->n_kv_heads * D * eb;
  if (cudaMemcpyAsync(q_dev, q_host, qb, cudaMemcpyHostToDevice, st) != cudaSuccess) return SANTA_ERR_CUDA;
  if (cudaMemcpyAsync(k_new_dev, k_new_host, kb, cudaMemcpyHostToDevice, st) != cudaSuccess) return SANTA_ERR_CUDA;
  if (cudaMemcpyAsync(v_new_dev, v_new_host, kb, cudaMemcpyHostToDevice, st) != cudaSuccess) return SANTA_ERR_CUDA;
  append_kv_kernel<<<dim3(g->n_kv_heads, g->batch), 128, 0, st>>>(K, V, k_new_dev, v_new_dev, kv_layout(g), seqlens,
                                                                  (int)D, (int)eb);
  if ((s = last_cuda()) != SANTA_OK) return s;
  if ((s = run_decode(a, SANTA_PATH_AUTO)) != SANTA_OK) return s;
  if (cudaMemcpyAsync(out_host, out_dev, qb, cudaMemcpyDeviceToHost, st) != cudaSuccess) return SANTA_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return SANTA_ERR_CUDA;
  return SANTA_OK;
}

santa_status santa_decode_step_host_packed(const santa_geometry* g, const void* qkv_host, void* qkv_dev, void* K,
                                           void* V, const int32_t* seqlens, int32_t S, int32_t mode, uint64_t seed,
                                           uint64_t offset, void* out_dev, void* out_host, void* ws, size_t ws_bytes,
                                           int32_t synchronize, void* stream) {
  santa_status s = validate_geometry(g);
  if (s != SANTA_OK) return s;
  if (!qkv_host || !qkv_dev || !out_host) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(qkv_dev)) return SANTA_ERR_ALIGNMENT;
  const size_t eb = elem_bytes(g->dtype), D = g->head_dim;
  const size_t qb = (size_t)g->batch * g->n_heads * D * eb, kb = (size_t)g->batch * g->n_kv_heads * D * eb;
  if ((qb % 16) || (kb % 16)) return SANTA_ERR_ALIGNMENT;  // k_new / v_new sub-buffers stay 16-B aligned
  // pinned host buffers are read / written by the kernels themselves (zero copy: no copy-engine
  // round trips); pageable ones go through cudaMemcpyAsync
  const void* qkv_alias = aligned16(qkv_host) ? pinned_alias(qkv_host) : nullptr;
  void* out_alias = aligned16(out_host) ? const_cast<void*>(pinned_alias(out_host)) : nullptr;
  // the whole decode validation runs before the first copy or launch (nothing is touched on error)
  DecodeArgs a;
  if ((s = prepare_decode(g, qkv_dev, K, V, seqlens, S, mode, seed, offset, out_alias ? out_alias : out_dev, nullptr,
                          ws, ws_bytes, nullptr, stream, SANTA_PATH_AUTO, &a)) != SANTA_OK)
    return s;
  if (!out_alias && !out_dev) return SANTA_ERR_INVALID_ARG;
  cudaStream_t st = a.st;
  char* dev = reinterpret_cast<char*>(qkv_dev);
  if (qkv_alias) {
    stage_append_kernel<<<dim3(g->n_kv_heads, g->batch), 128, 0, st>>>(
        reinterpret_cast<const uint4*>(qkv_alias), reinterpret_cast<uint4*>(dev), K, V, kv_layout(g), seqlens, (int)D,
        (int)eb, g->n_heads / g->n_kv_heads, g->n_heads);
  } else {
    if (cudaMemcpyAsync(dev, qkv_host, qb + 2 * kb, cudaMemcpyHostToDevice, st) != cudaSuccess) return SANTA_ERR_CUDA;
    append_kv_kernel<<<dim3(g->n_kv_heads, g->batch), 128, 0, st>>>(K, V, dev + qb, dev + qb + kb, kv_layout(g),
                                                                    seqlens, (int)D, (int)eb);
  }
  if ((s = last_cuda()) != SANTA_OK) return s;
  if ((s = run_decode(a, SANTA_PATH_AUTO)) != SANTA_OK) return s;
  if (!out_alias && cudaMemcpyAsync(out_host, out_dev, qb, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return SANTA_ERR_CUDA;
  if (synchronize && cudaStreamSynchronize(st) != cudaSuccess) return SANTA_ERR_CUDA;
  return SANTA_OK;
}

santa_status santa_philox_uniforms(uint64_t seed, uint64_t offset, int32_t tag, int32_t h_global, int32_t b_global,
                                   int32_t n, double* out, const uint32_t* ctr_key_host, uint32_t* raw_out,
                                   void* stream) {
  if (!out || n < 1) return SANTA_ERR_INVALID_ARG;
  uint4 ctr = make_uint4(0, 0, 0, 0);
  uint2 key = make_uint2(0, 0);
  if (ctr_key_host) {
    ctr = make_uint4(ctr_key_host[0], ctr_key_host[1], ctr_key_host[2], ctr_key_host[3]);
    key = make_uint2(ctr_key_host[4], ctr_key_host[5]);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  philox_test_kernel<<<(n + 255) / 256, 256, 0, st>>>(seed, offset, (uint32_t)tag, (uint32_t)h_global,
                                                      (uint32_t)b_global, n, out, ctr, key, raw_out);
  return last_cuda();
}

santa_status santa_read_error_flags(void* ws, uint32_t* flags_out, void* stream) {
  if (!ws || !flags_out) return SANTA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(ws) & 255u) return SANTA_ERR_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (cudaStreamSynchronize(st) != cudaSuccess) return SANTA_ERR_CUDA;
  if (cudaMemcpy(flags_out, ws, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return SANTA_ERR_CUDA;
  return SANTA_OK;
}

}  // extern "C"
