// santa_abi.cu -- host side of libsanta.so: argument validation, workspace layout,
// template dispatch and (PDL-chained) launches.  See include/santa.h for the contract.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>


#include "host.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges are no-ops unless a tool (nsys, ncu) attaches

using namespace santa;
using namespace santa_host;

namespace {

// one NVTX range per public entry point (a profiler timeline shows every ABI call by name)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
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

// local shard combine: (m_r, L_r) per (b, h) from the chunk stats, fp64
__global__ void shard_combine_kernel(const float2* __restrict__ cstats, const int32_t* __restrict__ seqlens,
                                     int H, int Cmax, int L, double* __restrict__ stats_out) {
  pdl_wait_primary();
  pdl_launch_dependents();  // a following PDL-launched score pass may set up meanwhile
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
  pdl_launch_dependents();  // the PDL-launched score pass sets up meanwhile (it waits for this grid)
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
__global__ void __launch_bounds__(128) stage_append_kernel(const uint4* __restrict__ qkv_h, uint4* __restrict__ q_dev,
                                                          void* K, void* V, KvLayout kv, const int32_t* seqlens, int D,
                                                          int eb, int G, int H) {
  const int kvh = blockIdx.x, b = blockIdx.y, Hkv = kv.n_kv_heads;
  const int row16 = D * eb / 16;                                 // 16-B words per row (<= 32)
  const size_t q16 = (size_t)gridDim.y * H * row16, k16 = (size_t)gridDim.y * Hkv * row16;
  const size_t qsrc = ((size_t)b * H + (size_t)kvh * G) * row16;
  const size_t ksrc = q16 + ((size_t)b * Hkv + kvh) * row16;
  // the PCIe reads first (launched with PDL: they overlap the preceding kernel's tail) ...
  const int nq = G * row16;                                      // <= 256 = 2 per thread
  uint4 qv[2], kr = make_uint4(0u, 0u, 0u, 0u), vr = kr;
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (threadIdx.x + 128 * r < nq) qv[r] = qkv_h[qsrc + threadIdx.x + 128 * r];
  if (threadIdx.x < row16) {
    kr = qkv_h[ksrc + threadIdx.x];
    vr = qkv_h[ksrc + k16 + threadIdx.x];
  }
  // ... every device write (q staging, cache slot) only after it has completed
  pdl_wait_primary();
  pdl_launch_dependents();  // the PDL-launched score pass sets up meanwhile (it waits for this grid)
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (threadIdx.x + 128 * r < nq) q_dev[qsrc + threadIdx.x + 128 * r] = qv[r];
  const int t = __ldg(seqlens + b) - 1;
  if (t < 0) return;
  const int64_t dst16 = kv.row(b, kvh, t, D) * eb / 16;
  if (threadIdx.x < row16) {
    reinterpret_cast<uint4*>(K)[dst16 + threadIdx.x] = kr;
    reinterpret_cast<uint4*>(V)[dst16 + threadIdx.x] = vr;
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
  // The score pass + sampler kernel everywhere since the round-2 changes (PDL-chained pass, 4-CTA-per-SM
  // sampler): config 2 20.1-21.1 vs 25.1-25.9 (step) / 28.9-29.2 us (tcgen05 step); batch 32 360-361 vs
  // 366 us for the tcgen05 step kernel at S = 64 and 381-386 vs 394 us at S = 256
  // (profiles/r02/v95_path_sweep_step_pdl.txt, v49_path_sweep.json).  The step kernels stay selectable.
  (void)g;
  (void)S;
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
  return "libsanta 0.4 sm_100a (santa_step_kernel: single-launch persistent step, tagged-word publication; santa_step_tc_kernel: tcgen05 score stage, TMEM accumulators; score_stream: TMA 128B-swizzle ring + mma.sync, interleaved, PDL-chained; sample_fast / sample_gather: thread-block clusters, 4-per-SM build for large batches; prop/flash: S^2ANTA-prop and -flash tile estimators; dense: TMA flash-decoding; bernoulli: bulk-copy ring + mma.sync with a 3-way bf16 weight split; peer_exchange: one-shot P2P collectives)";
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
  NvtxRange nvtx_("santa_decode_attention");
  return decode_common(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, nullptr, stream);
}

santa_status santa_decode_attention_path(const santa_geometry* g, const void* q, const void* K, const void* V,
                                         const int32_t* seqlens, int32_t S, int32_t mode, uint64_t seed,
                                         uint64_t offset, void* out, int32_t* idx_out, void* ws, size_t ws_bytes,
                                         int32_t path, void* stream) {
  NvtxRange nvtx_("santa_decode_attention_path");
  return decode_common(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, nullptr, stream,
                       path);
}

santa_status santa_decode_attention_profiled(const santa_geometry* g, const void* q, const void* K,
                                             const void* V, const int32_t* seqlens, int32_t S, int32_t mode,
                                             uint64_t seed, uint64_t offset, void* out, int32_t* idx_out,
                                             void* ws, size_t ws_bytes, void* const* events, void* stream) {
  NvtxRange nvtx_("santa_decode_attention_profiled");
  if (!events || !events[0] || !events[1] || !events[2]) return SANTA_ERR_INVALID_ARG;
  return decode_common(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, events, stream);
}

santa_status santa_score_phase(const santa_geometry* g, const void* q, const void* K, const int32_t* seqlens,
                               void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("santa_score_phase");
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
  NvtxRange nvtx_("santa_sample_phase");
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
  NvtxRange nvtx_("santa_decode_attention_prop");
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
  NvtxRange nvtx_("santa_decode_attention_flash");
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
  NvtxRange nvtx_("santa_dense_reference");
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
  NvtxRange nvtx_("santa_bernoulli_scores");
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
  NvtxRange nvtx_("santa_decode_attention_bernoulli");
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
  NvtxRange nvtx_("santa_seqshard_stats");
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
  NvtxRange nvtx_("santa_seqshard_sample_gather");
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
  NvtxRange nvtx_("santa_decode_step_host");
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
  NvtxRange nvtx_("santa_decode_step_host_packed");
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
    if (launch(stage_append_kernel, dim3(g->n_kv_heads, g->batch), dim3(128), 0, st, true,
               reinterpret_cast<const uint4*>(qkv_alias), reinterpret_cast<uint4*>(dev), K, V, kv_layout(g), seqlens,
               (int)D, (int)eb, g->n_heads / g->n_kv_heads, g->n_heads) != cudaSuccess)
      return SANTA_ERR_CUDA;
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

// decode step with the current token's KV append (fused into the score pass on the two-kernel path)
static santa_status decode_append(const santa_geometry* g, const void* q, void* K, void* V, const void* k_new,
                                  const void* v_new, const int32_t* seqlens, int32_t S, int32_t mode, uint64_t seed,
                                  uint64_t offset, void* out, int32_t* idx_out, void* ws, size_t ws_bytes,
                                  void* stream) {
  DecodeArgs a;
  santa_status s = prepare_decode(g, q, K, V, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, nullptr,
                                  stream, SANTA_PATH_AUTO, &a);
  if (s != SANTA_OK) return s;
  if (!k_new || !v_new) return SANTA_ERR_INVALID_ARG;
  if (!aligned16(k_new) || !aligned16(v_new)) return SANTA_ERR_ALIGNMENT;
  const int G = g->n_heads / g->n_kv_heads;
  if (auto_path(g, S) == SANTA_PATH_TWO_KERNEL && stream_eligible(g) && a.L.L == 64) {
    a.k_new = k_new;
    a.v_new = v_new;
    a.K_w = K;
    a.V_w = V;
    if ((s = dispatch<RunScore>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
    if ((s = dispatch<RunSample>(g->dtype, g->head_dim, G, a)) != SANTA_OK) return s;
    return last_cuda();
  }
  const int eb = elem_bytes(g->dtype);
  append_kv_kernel<<<dim3(g->n_kv_heads, g->batch), 128, 0, a.st>>>(K, V, k_new, v_new, kv_layout(g), seqlens,
                                                                    g->head_dim, eb);
  if ((s = last_cuda()) != SANTA_OK) return s;
  return run_decode(a, SANTA_PATH_AUTO);
}

santa_status santa_decode_attention_append(const santa_geometry* g, const void* q, void* K, void* V,
                                           const void* k_new, const void* v_new, const int32_t* seqlens, int32_t S,
                                           int32_t mode, uint64_t seed, uint64_t offset, void* out,
                                           int32_t* idx_out, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("santa_decode_attention_append");
  return decode_append(g, q, K, V, k_new, v_new, seqlens, S, mode, seed, offset, out, idx_out, ws, ws_bytes, stream);
}

static santa_status check_schedule(const santa_layer_schedule* sched) {
  if (!sched || !sched->S || sched->n_layers < 1) return SANTA_ERR_INVALID_ARG;
  for (int l = 0; l < sched->n_layers; ++l) {
    if (sched->S[l] < 1) return SANTA_ERR_EMPTY_BUDGET;
    if (sched->S[l] > kMaxBudget) return SANTA_ERR_UNSUPPORTED;
  }
  return SANTA_OK;
}

size_t santa_schedule_workspace_bytes(const santa_geometry* g, const santa_layer_schedule* sched) {
  if (validate_geometry(g) != SANTA_OK || check_schedule(sched) != SANTA_OK) return 0;
  size_t m = 0;
  for (int l = 0; l < sched->n_layers; ++l) m = std::max(m, layout(g, sched->S[l]).total);
  return m;
}

santa_status santa_decode_attention_layer(const santa_geometry* g, const santa_layer_schedule* sched, int32_t layer,
                                          const void* q, void* K, void* V, const void* k_new, const void* v_new,
                                          const int32_t* seqlens, int32_t mode, uint64_t seed, uint64_t offset,
                                          void* out, int32_t* idx_out, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("santa_decode_attention_layer");
  santa_status s = check_schedule(sched);
  if (s != SANTA_OK) return s;
  if (layer < 0 || layer >= sched->n_layers) return SANTA_ERR_INVALID_ARG;
  if ((k_new == nullptr) != (v_new == nullptr)) return SANTA_ERR_INVALID_ARG;
  const int32_t S = sched->S[layer];
  const uint64_t off = offset * (uint64_t)sched->n_layers + (uint64_t)layer;
  if (k_new)
    return decode_append(g, q, K, V, k_new, v_new, seqlens, S, mode, seed, off, out, idx_out, ws, ws_bytes, stream);
  return decode_common(g, q, K, V, seqlens, S, mode, seed, off, out, idx_out, ws, ws_bytes, nullptr, stream);
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
