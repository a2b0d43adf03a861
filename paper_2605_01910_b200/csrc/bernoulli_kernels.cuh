// bernoulli_kernels.cuh -- Bernoulli qK^T score stage (Eq. 5
// P:436-440, Eq. 6, App. C).  The paper implemented no kernel for it
// (P:47); this is new.
//
// bern_weights_kernel (one CTA per (b, kv-head), one thread per feature i):
//   mean-group (default): m_i = (1/G) sum_g |q_{g,i}|, norm = max_i m_i (reading #12),
//     a_i = m_i / norm, counts c_i from Philox tag 3 keyed by the GLOBAL kv-head,
//     stratified c_i = floor(B a_i) + 1[u_i < frac(B a_i)] (reading #11) or standard
//     c_i = #{n < B : u_{i,n} < a_i};  w_{g,i} = ((norm c_i / B) q_{g,i}) / m_i on the
//     selected set {c_i > 0, m_i > 0} (reading #14).
//   per-head ternary: norm_g = max_i |q_{g,i}|, counts from tag 2 keyed by the global head,
//     w_{g,i} = (norm_g / B) c_{g,i} sign(q_{g,i}); fetched set = union over the group (#15).
//   Every integer decision (a_i, floor, frac, compare) is taken in fp64 (the oracle takes the same decisions in fp64)
//   Output: fp32 weights [G][D], the compacted selected-feature list, the feature mask.
// bern_chunk_kernel (one CTA per 256-key chunk of (b, kv-head)): reads ONLY the selected
//   rows of the feature-major cache Kt, p_hat_g[k] = sum_{i in F} w_{g,i} Kt[i][k] (fp32
//   FMA; warp w takes features w, w+4, ...; lane takes 8 consecutive keys = one 16-B load),
//   writes scale * p_hat to `scores` if requested, then the same chunk max / exp2 / prefix
//   epilogue as the exact score pass -> the S^2ANTA sampler runs unchanged.
#pragma once
#include "common.cuh"
#include "philox.cuh"
#include "score_kernels.cuh"

namespace santa {

struct BernParams {
  const void* q;            // [B, H, D]
  const void* Kt;           // feature-major, see KtLayout
  const int32_t* seqlens;
  int B, H, Hkv, nB, stratified, mean_group;
  uint64_t seed, offset;
  int batch_offset, head_offset;
  float scale;              // natural-units scale for the scores output
  float* w;                 // [B*Hkv][G][D] fp32 weights
  int* sel;                 // [B*Hkv][D] selected features, count in sel_n
  int* sel_n;               // [B*Hkv]
  uint8_t* feature_mask;    // [B, Hkv or H, D] or NULL
  // chunk kernel
  const int32_t* page_table;
  int page_size, max_pages;
  float* scores;            // [B, H, score_stride] or NULL
  int score_stride;
  float* stash;
  float2* cstats;
  int Cmax, stash_stride;
  int sub64;                // 1: stats/stash per 64-key sub-chunk (Cmax/stash_stride of the L = 64 layout)
  uint32_t* tickets;
  uint32_t* flags;
  uint2* wfrag;             // [B*Hkv][D/16][3][32] bf16-part B fragments (bern_tma_kernel) or NULL
};

// B-fragment value of one bf16 part (0 = hi, 1 = mid, 2 = lo) of an fp32 weight: w = hi + mid + lo
// to 2^-24 |w| (bern_tma_kernel.cuh)
__device__ __forceinline__ uint16_t bern_weight_part(float w, int part) {
  __nv_bfloat16 h = __float2bfloat16_rn(w);
  if (part == 0) return __bfloat16_as_ushort(h);
  const float r1 = w - __bfloat162float(h);  // exact
  h = __float2bfloat16_rn(r1);
  if (part == 1) return __bfloat16_as_ushort(h);
  return __bfloat16_as_ushort(__float2bfloat16_rn(r1 - __bfloat162float(h)));
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(D) bern_weights_kernel(BernParams p) {
  __shared__ double sred[D / 32];
  __shared__ int sCount;
  const int kvh = blockIdx.x, b = blockIdx.y, i = threadIdx.x;
  const size_t unit = (size_t)b * p.Hkv + kvh;
  const T* q = reinterpret_cast<const T*>(p.q) + ((size_t)b * p.H + (size_t)kvh * G) * D;
  pdl_wait_primary();  // PDL launch: q (and the workspace) only after the preceding kernel completed
  if (i == 0) sCount = 0;
  double qd[G];
#pragma unroll
  for (int g = 0; g < G; ++g) qd[g] = (double)Elem<T>::to_f(q[g * D + i]);

  auto block_max = [&](double v) -> double {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((i & 31) == 0) sred[i >> 5] = v;
    __syncthreads();
    double r = sred[0];
#pragma unroll
    for (int k = 1; k < D / 32; ++k) r = fmax(r, sred[k]);
    return r;
  };
  auto counts = [&](double a, uint32_t tag, uint32_t id) -> int {
    PhiloxStream ps(p.seed, p.offset, tag, id, (uint32_t)(p.batch_offset + b));
    if (p.stratified) {
      const double Ba = (double)p.nB * a;
      const double fl = floor(Ba);
      return (int)fl + (ps.uniform((uint32_t)i) < (Ba - fl) ? 1 : 0);
    }
    int c = 0;
    for (int n = 0; n < p.nB; ++n) c += ps.uniform((uint32_t)(i * p.nB + n)) < a ? 1 : 0;
    return c;
  };

  float* w = p.w + unit * G * D;
  __shared__ float sWt[G * D];  // the weights and the selection again in shared memory: the fragment
  __shared__ int sSel[D];       // loop below reads them (from global it was a chain of L2 round trips)
  bool selected = false;
  if (p.mean_group) {
    double m = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g) m += fabs(qd[g]);
    m = m / (double)G;
    const double norm = block_max(m);
    int c = 0;
    if (norm > 0.0) c = counts(m / norm, kTagBernoulliGroup, (uint32_t)(p.head_offset / G + kvh));
    selected = c > 0 && m > 0.0;
    const double mhat = norm * (double)c / (double)p.nB;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float wv = selected ? (float)((mhat * qd[g]) / m) : 0.f;
      w[g * D + i] = wv;
      sWt[g * D + i] = wv;
    }
    if (p.feature_mask) p.feature_mask[unit * D + i] = selected ? 1 : 0;
  } else {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double norm = block_max(fabs(qd[g]));
      int c = 0;
      if (norm > 0.0) c = counts(fabs(qd[g]) / norm, kTagBernoulliHead, (uint32_t)(p.head_offset + kvh * G + g));
      const double sg = qd[g] > 0.0 ? 1.0 : (qd[g] < 0.0 ? -1.0 : 0.0);
      const float wv = c ? (float)((norm / (double)p.nB) * (double)c * sg) : 0.f;
      w[g * D + i] = wv;
      sWt[g * D + i] = wv;
      selected |= c > 0;
      if (p.feature_mask) p.feature_mask[((size_t)b * p.H + kvh * G + g) * D + i] = c > 0 ? 1 : 0;
    }
  }
  // compact the selected features in increasing i (deterministic order)
  __syncthreads();
  const unsigned bal = __ballot_sync(0xffffffffu, selected);
  __shared__ int sWarpCnt[D / 32];
  if ((i & 31) == 0) sWarpCnt[i >> 5] = __popc(bal);
  __syncthreads();
  int base = 0;
  for (int k = 0; k < (i >> 5); ++k) base += sWarpCnt[k];
  if (selected) {
    const int pos = base + __popc(bal & ((1u << (i & 31)) - 1u));
    p.sel[unit * D + pos] = i;
    sSel[pos] = i;
  }
  if (i == D - 1) {
    int tot = 0;
    for (int k = 0; k < D / 32; ++k) tot += sWarpCnt[k];
    p.sel_n[unit] = tot;
  }
  if (p.wfrag != nullptr) {
    // m16n8k16 B fragments of the weights in selection order (bern_tma_kernel): group kg of 16
    // selected features, part q of the 3-way bf16 split, lane (g, t) = (head g, features 2t, 2t+1
    // and 2t+8, 2t+9); heads >= G and features past |F| are 0.  sWt / sSel (shared) are
    // complete after the barrier.
    __syncthreads();
    int nsel = 0;
    for (int k = 0; k < D / 32; ++k) nsel += sWarpCnt[k];
    uint2* wf = p.wfrag + unit * (D / 16) * 96;
    for (int e = i; e < (D / 16) * 96; e += D) {
      const int kg = e / 96, q = (e / 32) % 3, ln = e % 32;
      const int g = ln >> 2, s0 = 16 * kg + 2 * (ln & 3);
      auto part = [&](int s) -> uint32_t {
        return (g < G && s < nsel) ? (uint32_t)bern_weight_part(sWt[g * D + sSel[s]], q) : 0u;
      };
      wf[e] = make_uint2(part(s0) | (part(s0 + 1) << 16), part(s0 + 8) | (part(s0 + 9) << 16));
    }
  }
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kScoreThreads, (sizeof(T) == 2 && G <= 4) ? 8 : 4) bern_chunk_kernel(BernParams p) {
  __shared__ __align__(16) float sS[G * kDenseChunk];
  __shared__ __align__(16) float sAcc[4][G][kDenseChunk];
  __shared__ float sW[G][D];
  __shared__ int sSel[D];
  pdl_wait_primary();
  pdl_launch_dependents();
  const int c = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  if (c == 0 && threadIdx.x == 0) {
    if (p.tickets) p.tickets[b * p.Hkv + kvh] = 0u;
    if (b == 0 && kvh == 0 && p.flags) *p.flags = 0u;
  }
  const int seqlen = __ldg(p.seqlens + b);
  const int chunk_start = c * kDenseChunk;
  const int n_valid = min(kDenseChunk, seqlen - chunk_start);
  const size_t unit = (size_t)b * p.Hkv + kvh;
  const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
  // stats/stash granularity: 64-key sub-chunks (sub64: the standard decode layout, 4 per CTA) or
  // the whole 256-key chunk
  const int cpc = p.sub64 ? kDenseChunk / 64 : 1;
  float2* cst = p.cstats + bh0 * p.Cmax + (size_t)c * cpc;
  if (n_valid <= 0) {
    if (threadIdx.x < G * cpc && (size_t)c * cpc + threadIdx.x % cpc < (size_t)p.Cmax)
      cst[(size_t)(threadIdx.x / cpc) * p.Cmax + threadIdx.x % cpc] = make_float2(-INFINITY, 0.f);
    if (p.scores && chunk_start < p.score_stride)
      for (int t = threadIdx.x; t < G * kDenseChunk; t += kScoreThreads) {
        const int k = chunk_start + t % kDenseChunk;
        if (k < p.score_stride) p.scores[(bh0 + t / kDenseChunk) * p.score_stride + k] = 0.f;
      }
    return;
  }
  const int nsel = p.sel_n[unit];
  for (int t = threadIdx.x; t < G * D; t += kScoreThreads) sW[t / D][t % D] = p.w[unit * G * D + t];
  for (int t = threadIdx.x; t < nsel; t += kScoreThreads) sSel[t] = p.sel[unit * D + t];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = p.page_table ? p.page_size : p.score_stride;  // contiguous: page = whole row
  const int kl = 8 * lane;            // this lane's 8 keys within the chunk
  const int t0 = chunk_start + kl;
  const int page = t0 / P, within = t0 - page * P;
  const int64_t phys = p.page_table ? (int64_t)__ldg(p.page_table + (int64_t)b * p.max_pages + page) : b;
  const T* Kt = reinterpret_cast<const T*>(p.Kt) + ((phys * p.Hkv + kvh) * D) * (int64_t)P + within;
  float acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[g][e] = 0.f;
  const bool live = kl < n_valid;
  // UF selected feature rows per warp in flight (16-B loads issued before any is consumed): one load
  // per lane per feature leaves ~6 KiB in flight per SM, far below what HBM needs (measured 0.37 of peak)
  constexpr int UF = (sizeof(T) == 2 && G <= 4) ? 4 : (sizeof(T) == 2 ? 8 : 4);  // rows in flight per warp
  for (int s0 = warp; s0 < nsel; s0 += 4 * UF) {
    uint4 r[UF][sizeof(T) == 2 ? 1 : 2];
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int s = s0 + 4 * u;
      if (live && s < nsel) {
        const T* src = Kt + (int64_t)sSel[s] * P;
        r[u][0] = ldg_stream(src);
        if constexpr (sizeof(T) == 4) r[u][1] = ldg_stream(src + 4);
      } else {
        r[u][0] = make_uint4(0u, 0u, 0u, 0u);
        if constexpr (sizeof(T) == 4) r[u][1] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int s = s0 + 4 * u;
      if (s >= nsel) break;
      const int i = sSel[s];
      float v[8];
      if constexpr (sizeof(T) == 2) {
        const uint32_t wv[4] = {r[u][0].x, r[u][0].y, r[u][0].z, r[u][0].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) { v[2 * e] = Elem<T>::lo(wv[e]); v[2 * e + 1] = Elem<T>::hi(wv[e]); }
      } else {
        v[0] = __uint_as_float(r[u][0].x); v[1] = __uint_as_float(r[u][0].y);
        v[2] = __uint_as_float(r[u][0].z); v[3] = __uint_as_float(r[u][0].w);
        v[4] = __uint_as_float(r[u][1].x); v[5] = __uint_as_float(r[u][1].y);
        v[6] = __uint_as_float(r[u][1].z); v[7] = __uint_as_float(r[u][1].w);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float wg = sW[g][i];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[g][e] = fmaf(wg, v[e], acc[g][e]);
      }
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < 8; ++e) sAcc[warp][g][kl + e] = acc[g][e];
  __syncthreads();
  const float sl2 = p.scale * kLog2e;
  for (int t = threadIdx.x; t < G * kDenseChunk; t += kScoreThreads) {
    const int g = t / kDenseChunk, k = t % kDenseChunk;
    const float ph = ((sAcc[0][g][k] + sAcc[1][g][k]) + sAcc[2][g][k]) + sAcc[3][g][k];
    const bool valid = k < n_valid;
    sS[p.sub64 ? ((k >> 6) * G + g) * 64 + (k & 63) : g * kDenseChunk + k] = valid ? ph * sl2 : -INFINITY;
    if (p.scores && chunk_start + k < p.score_stride)
      p.scores[(bh0 + g) * p.score_stride + chunk_start + k] = valid ? ph * p.scale : 0.f;
  }
  __syncthreads();
  if (p.stash) {
    if (p.sub64) {  // warp w: sub-chunk w with the L = 64 register epilogue (all G heads at once)
      const int sub_start = chunk_start + 64 * warp, n_sub = min(64, seqlen - sub_start);
      if (n_sub > 0)
        warp_chunk_epilogue<G>(sS + warp * G * 64, 64, n_sub, p.stash + bh0 * p.stash_stride + sub_start,
                               p.stash_stride, cst + warp, p.Cmax);
      else if (lane < G && (size_t)c * cpc + warp < (size_t)p.Cmax)
        cst[(size_t)lane * p.Cmax + warp] = make_float2(-INFINITY, 0.f);
    } else {
      chunk_epilogue<G>(sS, kDenseChunk, n_valid, warp, 4, p.stash + bh0 * p.stash_stride + chunk_start,
                        p.stash_stride, cst, p.Cmax);
    }
  }
}

__device__ __forceinline__ unsigned long long pack_f32x2(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void unpack_f32x2(unsigned long long v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
// d = a * b + c on both fp32 lanes of b / c, a broadcast (fma.rn.f32x2, sm_100 FFMA2)
__device__ __forceinline__ unsigned long long ffma2_bcast(float a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pack_f32x2(a, a)), "l"(b), "l"(c));
  return r;
}

// ---------------------------------------------------------------------------------------
// bern_stream_kernel: the Bernoulli score stage as a PERSISTENT stream (decode, 16-bit caches).
// The feature-major rows of the selected features are read key-block by key-block: work item =
// (unit, 2048 keys), warp w owns keys [256 w, 256 w + 256) of the block (lane l: 8 keys = one
// 16-B load per feature row) and loops over ALL selected features, so a warp's accumulators are
// final when its loop ends (no cross-warp reduction, no per-chunk CTA launch: the CTA-per-256-key
// kernel above ran ~16k short CTAs at 0.48-0.51 of peak).  Loads are software-pipelined UF
// features ahead in a register ring (UF * 512 B in flight per warp; 2 CTAs x 8 warps per SM).
// Items are interleaved over the grid; a CTA re-reads the weights / selection into shared memory
// when its next item belongs to another unit.  Epilogue: the L = 64 register
// epilogue of the exact score pass on each of the warp's four 64-key sub-chunks -> the sampler's
// stash / chunk stats layout (sub64), unchanged downstream.
constexpr int kBernStreamWarps = 8;
constexpr int kBernBlockKeys = kBernStreamWarps * 256;

template <typename T, int D, int G>
__global__ void __launch_bounds__(32 * kBernStreamWarps, 2) bern_stream_kernel(BernParams p, int items) {
  static_assert(sizeof(T) == 2, "16-bit caches");
  constexpr int UF = 16;
  __shared__ __align__(16) float sW[D][G];               // weights, feature-major
  __shared__ int sSel[D];
  __shared__ __align__(16) float sS[kBernStreamWarps][G * 64];  // one 64-key sub-chunk per warp at a time
  pdl_wait_primary();
  pdl_launch_dependents();
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.flags) *p.flags = 0u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = (p.score_stride + kBernBlockKeys - 1) / kBernBlockKeys;  // key blocks per unit (max_seqlen)
  // items interleaved over the grid (item t on CTA t % grid): the CTAs in flight cover whole units,
  // so every selected feature row is read along its full length by many CTAs at once (DRAM page
  // locality; a contiguous item range per CTA scattered the reads over ~27k open rows: 0.25 of peak)
  const int P = p.page_table ? p.page_size : p.score_stride;
  const float sl2 = p.scale * kLog2e;
  int cur_unit = -1, nsel = 0;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int unit = it / nblk, blk = it - unit * nblk;
    const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
    const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
    const int seqlen = __ldg(p.seqlens + b);
    const int blk_start = blk * kBernBlockKeys;
    if (blk_start >= seqlen) {  // whole block past the sequence: empty sub-chunk stats
      for (int t = threadIdx.x; t < G * (kBernBlockKeys / 64); t += blockDim.x) {
        const int c = blk_start / 64 + t % (kBernBlockKeys / 64);
        if (c < p.Cmax) p.cstats[(bh0 + t / (kBernBlockKeys / 64)) * p.Cmax + c] = make_float2(-INFINITY, 0.f);
      }
      continue;
    }
    if (unit != cur_unit) {  // (uniform over the CTA)
      __syncthreads();       // every warp is done with the previous unit's tables
      nsel = p.sel_n[unit];
      for (int t = threadIdx.x; t < G * D; t += blockDim.x) {
        const int g = t / D, i = t - g * D;
        sW[i][g] = p.w[(size_t)unit * G * D + t];
      }
      for (int t = threadIdx.x; t < nsel; t += blockDim.x) sSel[t] = p.sel[(size_t)unit * D + t];
      __syncthreads();
      cur_unit = unit;
    }
    // this lane's 8 keys
    const int k0 = blk_start + 256 * warp + 8 * lane;
    const bool live = k0 < seqlen;
    const int page = k0 / P, within = k0 - page * P;
    const int64_t phys = p.page_table ? (int64_t)__ldg(p.page_table + (int64_t)b * p.max_pages + page) : b;
    const T* Kt = reinterpret_cast<const T*>(p.Kt) + ((phys * p.Hkv + kvh) * D) * (int64_t)P + within;
    unsigned long long acc2[G][4];  // fp32 pairs: keys (2e, 2e+1)
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc2[g][e] = 0ull;
    // two batches of UB feature rows in flight: issue batch k+1, then consume batch k (the loads of a
    // batch complete on one scoreboard -- a 16-deep single ring shared scoreboards between old and
    // freshly issued loads and waited a full DRAM latency per row: 0.25 of peak, ncu long_scoreboard)
    constexpr int UB = UF / 2;
    uint4 ra[UB], rb[UB];
    auto issue = [&](uint4 (&r)[UB], int s0) {
#pragma unroll
      for (int u = 0; u < UB; ++u)
        r[u] = (live && s0 + u < nsel) ? ldg_stream(Kt + (int64_t)sSel[s0 + u] * P) : make_uint4(0u, 0u, 0u, 0u);
    };
    // the FMAs as packed fp32x2 (FFMA2, sm_100: two keys per instruction, the weight broadcast; each
    // lane is an IEEE fma, bit-identical to fmaf): the kernel was issue-bound on 32 FFMA per row segment
    auto consume = [&](const uint4 (&r)[UB], int s0) {
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int s = s0 + u;
        if (s >= nsel) break;
        const int i = sSel[s];
        const float4 w4 = *reinterpret_cast<const float4*>(&sW[i][0]);
        const float wg[4] = {w4.x, w4.y, w4.z, w4.w};
        const uint32_t wv[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
        unsigned long long v2[4];  // keys (2e, 2e+1) as an fp32 pair
#pragma unroll
        for (int e = 0; e < 4; ++e) v2[e] = pack_f32x2(Elem<T>::lo(wv[e]), Elem<T>::hi(wv[e]));
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float wgt = G <= 4 ? wg[g] : sW[i][g];
#pragma unroll
          for (int e = 0; e < 4; ++e) acc2[g][e] = ffma2_bcast(wgt, v2[e], acc2[g][e]);
        }
      }
    };
    issue(ra, 0);
    for (int s0 = 0; s0 < nsel; s0 += UF) {
      issue(rb, s0 + UB);
      consume(ra, s0);
      issue(ra, s0 + UF);
      consume(rb, s0 + UB);
    }
    float acc[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < 4; ++e) unpack_f32x2(acc2[g][e], acc[g][2 * e], acc[g][2 * e + 1]);
    // epilogue: the warp's 4 sub-chunks of 64 keys, each through smem [G][64]
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
      const int sub_start = blk_start + 256 * warp + 64 * sub;
      const int n_sub = min(64, seqlen - sub_start);
      // lanes 8 sub .. 8 sub + 7 hold this sub-chunk's keys
      if ((lane >> 3) == sub) {
        const int kk = 8 * (lane & 7);
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const bool valid = kk + e < n_sub;
            sS[warp][g * 64 + kk + e] = valid ? acc[g][e] * sl2 : -INFINITY;
            if (p.scores && sub_start + kk + e < p.score_stride)
              p.scores[(bh0 + g) * p.score_stride + sub_start + kk + e] = valid ? acc[g][e] * p.scale : 0.f;
          }
      }
      __syncwarp();
      const int c = sub_start / 64;
      if (n_sub > 0) {
        if (p.stash)
          warp_chunk_epilogue<G>(sS[warp], 64, n_sub, p.stash + bh0 * p.stash_stride + sub_start, p.stash_stride,
                                 p.cstats + bh0 * p.Cmax + c, p.Cmax);
      } else if (lane < G && c < p.Cmax) {
        p.cstats[(bh0 + lane) * p.Cmax + c] = make_float2(-INFINITY, 0.f);
      }
      __syncwarp();
    }
  }
}

}  // namespace santa
