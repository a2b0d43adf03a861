// sample_kernels.cuh -- combine + sampler + gather-add of the SANTA decode hot path
// (SURVEY sec. 8(a) rows a3-a6).
//
// sample_item() handles one (batch b, query head h, split `rank` of CS): the strata
// m in [S*rank/CS, S*(rank+1)/CS) of that head.  Steps:
//  a4 thresholds (before griddepcontrol.wait, overlapping the score pass when launched with
//     PDL): Philox4x32-10, T_m in fp64 exactly as the oracle (readings #1-#3).
//  a3 combine: the head's chunk stats are loaded in one round trip; m* = max_c m_c,
//     W_c = 2^(m_c - m*) l_c (fp64), block-wide fp64 scan -> F_c = sum_{c'<=c} W / Z, clamped
//     to 1 from the last positive chunk on (reading #5); the in-chunk rescale Z l_c / W_c is kept
//     per chunk.  (The LSE merge of Alg. prop-budgets P:1606-1607 / flash-k2 P:1701, in fp64.)
//  a5 inverse CDF: c = min{c : F_c > T} by binary search in shared memory (thread per sample),
//     then k = min{k : P_c[k] > t}, t = (T - F_{c-1}) Z 2^(m* - m_c), J = c L + k (P:699,
//     reading #4): a HALF-WARP per sample loads the chunk's 256-B prefix block coalesced and
//     counts P[k] <= rd(t) with ballots (exact, reading #21).
//  a6 gather-add: the same 16 lanes then load the sample's V row (16 B each) and add it;
//     8 samples in flight per half-warp; fixed-order reduction over half-warps -> the CTA's
//     partial sum (1/S and the cast are applied by the caller; "adds only",
//     Table).  V rows shared by the G heads of a group are deduplicated by the L2.
//  Sequence-sharded mode (stats_all != NULL, reading #18): the global threshold T is first
//  located in the shard CDF built from every rank's (m_r, L_r); strata outside this rank's
//  [F_{r-1}, F_r) are skipped, owned ones are re-normalised to the local distribution.
//
// sample_gather_kernel: grid (H*CS, B); the CS CTAs of a head form one thread-block cluster
// and sum their partials through distributed shared memory in fixed rank order.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "philox.cuh"

namespace santa {

constexpr int kSampleThreads = 256;
constexpr int kMaxBudget = 4096;  // S limit (shared-memory sample tables)

struct SampleParams {
  const float* stash;
  const float2* cstats;
  int Cmax, L, stash_stride;
  const void* V;
  KvLayout kv;
  const int32_t* seqlens;
  int B, H, Hkv, S, mode;
  uint64_t seed, offset;
  int batch_offset, head_offset;
  void* out;                    // [B, H, D] dtype T (standard mode)
  float* out_f32;               // [B, H, D] fp32 (seq-shard partial mode) -- used if non-NULL
  int32_t* idx_out;             // [B, H, S] or NULL
  uint32_t* flags;
  // sequence sharding
  const double* stats_all;      // [world, B, H, 2] or NULL
  int rank, world;
  const int32_t* token_offset;  // [B] or NULL
  int cluster;                  // CTAs per head (thread-block cluster size / splits)
  float* split_partial;         // fused kernel: [B*H*cluster][D] scratch
  unsigned long long* trace;    // NULL in the library; tools/microbench_sample.cu phase timing
};

#define SANTA_TRACE(i)                                                   \
  if (p.trace && threadIdx.x == 0 && rank == 0)                          \
  p.trace[((size_t)b * p.H + h) * 16 + (i)] = gtimer()

// min{k in [0, n) : P[k] > t} for a non-decreasing fp32 array P (n if none), by one thread (no
// warp collectives).  Because P[k] is fp32, P[k] > t  <=>  P[k] > rd(t) (t rounded toward -inf
// to fp32), so passing tf = rd(t) decides the fp64 comparison exactly.  Used for chunks longer
// than 64 and for the rare rounding fallback; the L = 64 fast path uses half-warp ballots.
__device__ __forceinline__ int thread_chunk_search(const float* __restrict__ P, int n, float tf) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldcg(P + mid) > tf) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// block-wide reductions for any blockDim.x that is a multiple of 32 (<= 1024)
__device__ __forceinline__ float block_max_f(float v, float* sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  float r = sred[0];
  for (int w = 1; w < nw; ++w) r = fmaxf(r, sred[w]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ int block_max_i(int v, int* sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  int r = sred[0];
  for (int w = 1; w < nw; ++w) r = max(r, sred[w]);
  __syncthreads();
  return r;
}

// block-wide exclusive scan of one double per thread; *total receives the sum
__device__ __forceinline__ double block_excl_scan_d(double v, double* sred, double* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double incl = warp_incl_scan_d(v, lane);
  if (lane == 31) sred[warp] = incl;
  __syncthreads();
  double off = 0.0, tot = 0.0;
  for (int w = 0; w < nw; ++w) {
    const double x = sred[w];
    if (w < warp) off += x;
    tot += x;
  }
  __syncthreads();
  *total = tot;
  return off + incl - v;
}

// Skewed index of chunk c in sample_item's per-chunk fp64 tables: thread t owns the contiguous chunks
// [t per, t per + per), so unskewed 8-B entries put a warp's 32 threads in one bank group (a 32-way
// conflict per access -- 19.5 us of fp64 CDF build at 4096 chunks, config 4 phase 2 at R = 2); one pad
// entry per 16 spreads them.
__host__ __device__ __forceinline__ int cskew(int c) { return c + (c >> 4); }

// Shared-memory bytes sample_item needs for a CTA of nthreads threads.
__host__ __device__ inline size_t sample_smem_bytes(int Cmax, int S_local, int D, int nthreads) {
  return (size_t)cskew(Cmax) * 16 + 16 + (size_t)S_local * 16 + (size_t)(nthreads / 16 + 1) * D * 4 + 64;
}

// a5 (part 2) + a6 for the Sl samples of one work item whose chunk sChunk[m] (-1: not sampled
// here) and in-chunk threshold sTl[m] are in shared memory: a HALF-WARP per sample finds
// k = min{k : P_c[k] > sTl[m]} in the chunk's prefix block (ballots, L = 64; binary search
// otherwise), writes idx_out[bh, m_lo + m], then loads and adds the V row; the half-warps'
// sums are reduced in fixed order into sPart [D] (unscaled).  All threads call it.
// kW: each sample's row is scaled by sWt[m] (S^2ANTA-flash merge weights); idx rows are
// idx_stride long (default S).
template <typename T, int D, bool kW, int U>
__device__ __forceinline__ void gather_chunk_rows_u(const SampleParams& p, int b, int h, int rank, int kvh, size_t bh,
                                                    int Sl, int m_lo, int seqlen, const int* sChunk,
                                                    const float* sTl, float* sRed, float* sPart, const float* sWt,
                                                    int idx_stride) {
  const int NT = blockDim.x, NHW = NT >> 4;
  const int tid = threadIdx.x;
  const int S = idx_stride < 0 ? p.S : idx_stride;
  constexpr int EB = (int)sizeof(T);
  constexpr int VCH = D * EB / 16;                  // 16-B chunks per V row
  constexpr int NCH = (VCH + 15) / 16;              // chunks per lane
  constexpr int EPC = 16 / EB;                      // elements per chunk
  const int hw = tid >> 4, l = tid & 15;
  const unsigned hmask = 0xffffu << (threadIdx.x & 16);
  float acc[NCH][EPC];
#pragma unroll
  for (int q = 0; q < NCH; ++q)
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[q][e] = 0.f;
  const T* Vb = reinterpret_cast<const T*>(p.V);
  const float* Pbase = p.stash + bh * p.stash_stride;
  // V row address: contiguous caches hoist the (b, kv-head) base (one multiply-add per row; the
  // generic paged/contiguous KvLayout::row() inlined per sample serialised the loads' issue)
  const T* vbase = p.kv.page_table ? Vb : Vb + ((int64_t)b * p.kv.n_kv_heads + kvh) * p.kv.page_size * D;
  auto vrow = [&](int t) -> const T* {
    return p.kv.page_table ? Vb + p.kv.row(b, kvh, t, D) : vbase + (int64_t)t * D;
  };
  const int tok0 = p.token_offset ? __ldg(p.token_offset + b) : 0;
  // warp-uniform trip count: warp w walks sample pairs 2w, 2w+1 (+ NHW per u); the full-mask
  // ballots below must be reached by both half-warps
  for (int mw = 2 * (tid >> 5); mw < Sl; mw += NHW * U) {
    const int m0 = mw + (hw & 1);
    int jj[U];
    float4 pv[U];
    int cc[U], nn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + u * NHW;
      cc[u] = m < Sl ? sChunk[m] : -1;
      nn[u] = cc[u] >= 0 ? min(p.L, seqlen - cc[u] * p.L) : 0;
      pv[u] = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
      if (cc[u] >= 0 && p.L == 64 && 4 * l < nn[u])
        pv[u] = ldcg_f4(reinterpret_cast<const float4*>(Pbase + (size_t)cc[u] * p.L) + l);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // in-chunk index k = min{k : P[k] > tf} = #{k : P[k] <= tf} (P non-decreasing; inactive samples
      // and keys beyond the sequence load P = +inf).  L = 64, branch-free: one ballot over every
      // lane's last value (lane j holds keys 4j..4j+3) + the crossing lane's own count.
      const int m = m0 + u * NHW;
      const bool on = cc[u] >= 0;
      const float tf = on ? sTl[m] : -INFINITY;
      const float4 v = pv[u];
      int k;
      if (p.L == 64) {
        const int full_lanes = __popc(__ballot_sync(0xffffffffu, v.w <= tf) & hmask);
        const int own = (v.x <= tf) + (v.y <= tf) + (v.z <= tf) + (v.w <= tf);
        const int cross = __shfl_sync(0xffffffffu, own, (tid & 16) + min(full_lanes, 15));
        k = full_lanes < 16 ? 4 * full_lanes + cross : 64;
        // rounding put tf at/after the chunk's total: the first key reaching the total (the last
        // positive-mass key); the total P[n-1] sits in lane (n-1)/4, component (n-1)%4
        if (__any_sync(0xffffffffu, on && k >= nn[u])) {
          const int ln = max(nn[u] - 1, 0);
          const int src = (tid & 16) + (ln >> 2);
          const float tx = __shfl_sync(0xffffffffu, v.x, src), ty = __shfl_sync(0xffffffffu, v.y, src);
          const float tz = __shfl_sync(0xffffffffu, v.z, src), tw = __shfl_sync(0xffffffffu, v.w, src);
          const float tot = (ln & 3) == 0 ? tx : (ln & 3) == 1 ? ty : (ln & 3) == 2 ? tz : tw;
          const int fl2 = __popc(__ballot_sync(0xffffffffu, v.w < tot) & hmask);
          const int own2 = (v.x < tot) + (v.y < tot) + (v.z < tot) + (v.w < tot);
          const int cross2 = __shfl_sync(0xffffffffu, own2, (tid & 16) + min(fl2, 15));
          if (on && k >= nn[u]) k = fl2 < 16 ? 4 * fl2 + cross2 : nn[u] - 1;
        }
      } else {
        k = 0;
        if (on) {
          const float* P = Pbase + (size_t)cc[u] * p.L;
          k = thread_chunk_search(P, nn[u], tf);
          if (k >= nn[u]) k = thread_chunk_search(P, nn[u], nextafterf(__ldcg(P + nn[u] - 1), -INFINITY));
        }
      }
      jj[u] = on ? cc[u] * p.L + min(k, nn[u] - 1) : -1;
      if (on && l == 0 && p.idx_out) p.idx_out[bh * S + m_lo + m] = jj[u] + tok0;
      if (!on && m < Sl && l == 0 && p.idx_out) p.idx_out[bh * S + m_lo + m] = -1;  // another shard's stratum
    }
    if (mw == 0) SANTA_TRACE(8);  // indices known (stash loaded, ballots done)
    uint4 raw[U][NCH];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        const int ch = l + 16 * q;
        raw[u][q] = (jj[u] >= 0 && ch < VCH) ? ldg_nc(vrow(jj[u]) + ch * EPC) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float wt = 1.f;
      if constexpr (kW) wt = jj[u] >= 0 ? sWt[m0 + u * NHW] : 0.f;
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        if constexpr (EB == 2) {
          const uint32_t w[4] = {raw[u][q].x, raw[u][q].y, raw[u][q].z, raw[u][q].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if constexpr (kW) {
              acc[q][2 * e] = fmaf(wt, Elem<T>::lo(w[e]), acc[q][2 * e]);
              acc[q][2 * e + 1] = fmaf(wt, Elem<T>::hi(w[e]), acc[q][2 * e + 1]);
            } else {
              acc[q][2 * e] += Elem<T>::lo(w[e]);
              acc[q][2 * e + 1] += Elem<T>::hi(w[e]);
            }
          }
        } else {
          acc[q][0] = fmaf(wt, __uint_as_float(raw[u][q].x), acc[q][0]);
          acc[q][1] = fmaf(wt, __uint_as_float(raw[u][q].y), acc[q][1]);
          acc[q][2] = fmaf(wt, __uint_as_float(raw[u][q].z), acc[q][2]);
          acc[q][3] = fmaf(wt, __uint_as_float(raw[u][q].w), acc[q][3]);
        }
      }
    }
  }
  SANTA_TRACE(9);  // V rows gathered and added (thread 0)
  // deterministic reduction over the half-warps (fixed order)
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    const int ch = l + 16 * q;
    if (ch < VCH)
#pragma unroll
      for (int e = 0; e < EPC; ++e) sRed[hw * D + ch * EPC + e] = acc[q][e];
  }
  __syncthreads();
  SANTA_TRACE(6);
  for (int d = tid; d < D; d += NT) {
    float s = 0.f;
    for (int r = 0; r < NHW; ++r) s += sRed[r * D + d];
    sPart[d] = s;
  }
  __syncthreads();
}

// Two-phase form of gather_chunk_rows_u for register-capped builds (4 CTAs per SM): phase 1 finds
// the in-chunk index of U samples per half-warp per round (their prefix blocks in flight together)
// and parks J in sChunk; phase 2 loads U V rows per round.  With 16 samples per half-warp this is
// 2 + 2 dependent memory round trips instead of 4 x (prefix block -> V row) = 8 for the fused loop
// at U = 4 -- and only one U-deep buffer is live at a time.  Same ballots, same fixed-order sums.
template <typename T, int D, bool kW, int U, int U2 = U>
__device__ __forceinline__ void gather_chunk_rows_2ph(const SampleParams& p, int b, int h, int rank, int kvh, size_t bh,
                                                      int Sl, int m_lo, int seqlen, int* sChunk, const float* sTl,
                                                      float* sRed, float* sPart, const float* sWt, int idx_stride) {
  const int NT = blockDim.x, NHW = NT >> 4;
  const int tid = threadIdx.x;
  const int S = idx_stride < 0 ? p.S : idx_stride;
  constexpr int EB = (int)sizeof(T);
  constexpr int VCH = D * EB / 16;
  constexpr int NCH = (VCH + 15) / 16;
  constexpr int EPC = 16 / EB;
  const int hw = tid >> 4, l = tid & 15;
  const unsigned hmask = 0xffffu << (threadIdx.x & 16);
  const float* Pbase = p.stash + bh * p.stash_stride;
  const int tok0 = p.token_offset ? __ldg(p.token_offset + b) : 0;
  // ---- phase 1: J of every sample (L = 64 ballots; binary search for longer chunks) ----
  for (int mw = 2 * (tid >> 5); mw < Sl; mw += NHW * U) {
    const int m0 = mw + (hw & 1);
    int cc[U], nn[U];
    float4 pv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + u * NHW;
      cc[u] = m < Sl ? sChunk[m] : -1;
      nn[u] = cc[u] >= 0 ? min(p.L, seqlen - cc[u] * p.L) : 0;
      pv[u] = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
      if (cc[u] >= 0 && p.L == 64 && 4 * l < nn[u])
        pv[u] = ldcg_f4(reinterpret_cast<const float4*>(Pbase + (size_t)cc[u] * p.L) + l);
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + u * NHW;
      const bool on = cc[u] >= 0;
      const float tf = on ? sTl[m] : -INFINITY;
      const float4 v = pv[u];
      int k;
      if (p.L == 64) {
        const int full_lanes = __popc(__ballot_sync(0xffffffffu, v.w <= tf) & hmask);
        const int own = (v.x <= tf) + (v.y <= tf) + (v.z <= tf) + (v.w <= tf);
        const int cross = __shfl_sync(0xffffffffu, own, (tid & 16) + min(full_lanes, 15));
        k = full_lanes < 16 ? 4 * full_lanes + cross : 64;
        if (__any_sync(0xffffffffu, on && k >= nn[u])) {
          const int ln = max(nn[u] - 1, 0);
          const int src = (tid & 16) + (ln >> 2);
          const float tx = __shfl_sync(0xffffffffu, v.x, src), ty = __shfl_sync(0xffffffffu, v.y, src);
          const float tz = __shfl_sync(0xffffffffu, v.z, src), tw = __shfl_sync(0xffffffffu, v.w, src);
          const float tot = (ln & 3) == 0 ? tx : (ln & 3) == 1 ? ty : (ln & 3) == 2 ? tz : tw;
          const int fl2 = __popc(__ballot_sync(0xffffffffu, v.w < tot) & hmask);
          const int own2 = (v.x < tot) + (v.y < tot) + (v.z < tot) + (v.w < tot);
          const int cross2 = __shfl_sync(0xffffffffu, own2, (tid & 16) + min(fl2, 15));
          if (on && k >= nn[u]) k = fl2 < 16 ? 4 * fl2 + cross2 : nn[u] - 1;
        }
      } else {
        k = 0;
        if (on) {
          const float* P = Pbase + (size_t)cc[u] * p.L;
          k = thread_chunk_search(P, nn[u], tf);
          if (k >= nn[u]) k = thread_chunk_search(P, nn[u], nextafterf(__ldcg(P + nn[u] - 1), -INFINITY));
        }
      }
      const int j = on ? cc[u] * p.L + min(k, nn[u] - 1) : -1;
      if (l == 0 && m < Sl) {
        sChunk[m] = j;   // this half-warp's own sample: no other thread reads it before the barrier
        if (p.idx_out) p.idx_out[bh * S + m_lo + m] = on ? j + tok0 : -1;
      }
    }
  }
  __syncthreads();
  SANTA_TRACE(8);  // every J known (prefix blocks loaded, ballots done)
  // ---- phase 2: V rows, U per half-warp in flight ----
  float acc[NCH][EPC];
#pragma unroll
  for (int q = 0; q < NCH; ++q)
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[q][e] = 0.f;
  const T* Vb = reinterpret_cast<const T*>(p.V);
  const T* vbase = p.kv.page_table ? Vb : Vb + ((int64_t)b * p.kv.n_kv_heads + kvh) * p.kv.page_size * D;
  for (int m0 = hw; m0 < Sl; m0 += NHW * U2) {
    uint4 raw[U2][NCH];
    float wt[U2];
#pragma unroll
    for (int u = 0; u < U2; ++u) {
      const int m = m0 + u * NHW;
      const int j = m < Sl ? sChunk[m] : -1;
      wt[u] = 1.f;
      if constexpr (kW) wt[u] = j >= 0 ? sWt[m] : 0.f;
      const T* row = j >= 0 ? (p.kv.page_table ? Vb + p.kv.row(b, kvh, j, D) : vbase + (int64_t)j * D) : nullptr;
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        const int ch = l + 16 * q;
        raw[u][q] = (j >= 0 && ch < VCH) ? ldg_nc(row + ch * EPC) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int u = 0; u < U2; ++u)
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        if constexpr (EB == 2) {
          const uint32_t w[4] = {raw[u][q].x, raw[u][q].y, raw[u][q].z, raw[u][q].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if constexpr (kW) {
              acc[q][2 * e] = fmaf(wt[u], Elem<T>::lo(w[e]), acc[q][2 * e]);
              acc[q][2 * e + 1] = fmaf(wt[u], Elem<T>::hi(w[e]), acc[q][2 * e + 1]);
            } else {
              acc[q][2 * e] += Elem<T>::lo(w[e]);
              acc[q][2 * e + 1] += Elem<T>::hi(w[e]);
            }
          }
        } else {
          acc[q][0] = fmaf(wt[u], __uint_as_float(raw[u][q].x), acc[q][0]);
          acc[q][1] = fmaf(wt[u], __uint_as_float(raw[u][q].y), acc[q][1]);
          acc[q][2] = fmaf(wt[u], __uint_as_float(raw[u][q].z), acc[q][2]);
          acc[q][3] = fmaf(wt[u], __uint_as_float(raw[u][q].w), acc[q][3]);
        }
      }
  }
  SANTA_TRACE(9);  // V rows gathered and added (thread 0)
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    const int ch = l + 16 * q;
    if (ch < VCH)
#pragma unroll
      for (int e = 0; e < EPC; ++e) sRed[hw * D + ch * EPC + e] = acc[q][e];
  }
  __syncthreads();
  SANTA_TRACE(6);
  for (int d = tid; d < D; d += NT) {
    float s = 0.f;
    for (int r = 0; r < NHW; ++r) s += sRed[r * D + d];
    sPart[d] = s;
  }
  __syncthreads();
}

// U = samples in flight per half-warp.  U = 4 when one pass covers the work item (config 2: 4 per
// half-warp): the unrolled U = 8 body is twice the code, half of it predicated off, and its
// instruction fetch was the kernel's top stall (ncu `no_instructions` 52 %; sample phase 9.1 -> 8.1
// us); U = 8 otherwise (flash at S = 2048: 36.9 vs 40.6 us with U = 4).
template <typename T, int D, bool kW = false, int UMAX = 8>
__device__ __forceinline__ void gather_chunk_rows(const SampleParams& p, int b, int h, int rank, int kvh, size_t bh,
                                                  int Sl, int m_lo, int seqlen, const int* sChunk,
                                                  const float* sTl, float* sRed, float* sPart,
                                                  const float* sWt = nullptr, int idx_stride = -1) {
  if (UMAX <= 4 || Sl <= 4 * (int)(blockDim.x >> 4))
    gather_chunk_rows_u<T, D, kW, 4>(p, b, h, rank, kvh, bh, Sl, m_lo, seqlen, sChunk, sTl, sRed, sPart, sWt,
                                     idx_stride);
  else
    gather_chunk_rows_u<T, D, kW, 8>(p, b, h, rank, kvh, bh, Sl, m_lo, seqlen, sChunk, sTl, sRed, sPart, sWt,
                                     idx_stride);
}

// One (b, h, split) work item.  Leaves the CTA's partial sum sum_{own m} V_{J_m} (fp32, not yet
// scaled by 1/S) in the returned shared array [D]; the caller reduces/scales/writes it.  All
// threads of the block must call it.  Empty sequences (seqlen < 1) give a zero partial, idx -1
// and the workspace flag.
template <typename T, int D, int G, int UMAX = 8>
__device__ float* sample_item(const SampleParams& p, int b, int h, int rank, int CS, unsigned char* smem_raw) {
  const int NT = blockDim.x, NW = NT >> 5, NHW = NT >> 4;
  const int kvh = h / G;
  const int tid = threadIdx.x;
  const size_t bh = (size_t)b * p.H + h;
  const int S = p.S;                                    // global budget (thresholds, 1/S)
  const int m_lo = (int)((long long)S * rank / CS), m_hi = (int)((long long)S * (rank + 1) / CS);
  const int Sl = m_hi - m_lo;                           // strata owned by this item
  const int Slmax = (S + CS - 1) / CS;
  const int CmaxS = cskew(p.Cmax) + 1;                  // skewed table length (index cskew(c))
  double* sF = reinterpret_cast<double*>(smem_raw);     // [CmaxS] chunk CDF
  double* sT = sF + CmaxS;                              // [Slmax] thresholds
  float2* sC = reinterpret_cast<float2*>(sT + Slmax);   // [CmaxS] chunk stats, then rescale (double)
  int* sChunk = reinterpret_cast<int*>(sC + CmaxS);     // [Slmax]
  float* sTl = reinterpret_cast<float*>(sChunk + Slmax);  // [Slmax]
  float* sRed = sTl + Slmax;                            // [NHW][D]
  float* sPart = sRed + NHW * D;                        // [D]
  __shared__ double sred_d[32];
  __shared__ float sred_f[32];
  __shared__ int sred_i[32];
  __shared__ double sTlo, sThi, sTscale;
  __shared__ int sOwnAny;
  (void)NW;

  SANTA_TRACE(0);
  // ---- a4: thresholds (independent of the score pass) ---------------------------------------
  {
    PhiloxStream ps(p.seed, p.offset, kTagValueSampler, (uint32_t)(p.head_offset + h), (uint32_t)(p.batch_offset + b));
    for (int i = tid; i < Sl; i += NT) sT[i] = sample_threshold(p.mode, m_lo + i, S, ps);
  }
  SANTA_TRACE(1);
  pdl_wait_primary();
  pdl_launch_dependents();  // the next kernel (waiting on this grid itself) may set up meanwhile
  SANTA_TRACE(2);

  const int seqlen = __ldg(p.seqlens + b);
  if (seqlen < 1) {  // empty distribution: zero partial, flag, no sampling
    for (int d = tid; d < D; d += NT) sPart[d] = 0.f;
    if (rank == 0 && tid == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    if (p.idx_out)
      for (int i = tid; i < Sl; i += NT) p.idx_out[bh * S + m_lo + i] = -1;
    __syncthreads();
    return sPart;
  }
  const int nC = (seqlen + p.L - 1) / p.L;

  // ---- a3: chunk stats -> fp64 chunk CDF ------------------------------------------------------
  // thread t owns the contiguous chunks [t*per, t*per + per); for <= 8 per thread (nC <= 8 NT) they
  // are loaded straight into registers (one round trip), W_c = 2^(m_c - m*) l_c with the power in fp32
  // (ex2.approx, 2 ulp -- the fp32 scores already carry errors of that order) and the sums, the CDF
  // and the in-chunk rescale in fp64 (as the step kernel, reading #24)
  const float2* cs = p.cstats + bh * p.Cmax;
  const int per = (nC + NT - 1) / NT;
  const int c0 = min(tid * per, nC), c1 = min(c0 + per, nC);
  constexpr int kCPT = 8;
  double part = 0.0;
  int lastpos = -1;
  if (per <= kCPT) {
    float2 st[kCPT];
#pragma unroll
    for (int i = 0; i < kCPT; ++i) st[i] = (c0 + i < c1) ? __ldcg(cs + c0 + i) : make_float2(-INFINITY, 0.f);
    float mloc = -INFINITY;
#pragma unroll
    for (int i = 0; i < kCPT; ++i) mloc = fmaxf(mloc, st[i].x);
    const float mstar = block_max_f(mloc, sred_f);
    SANTA_TRACE(3);
#pragma unroll
    for (int i = 0; i < kCPT; ++i) {
      if (c0 + i >= c1) break;
      const float w32 = st[i].y > 0.f ? ex2(st[i].x - mstar) : 0.f;  // 2^(m_c - m*)
      const double w = (double)w32 * (double)st[i].y;
      sF[cskew(c0 + i)] = w;
      // in-chunk rescale Z 2^(m* - m_c) = Z l_c / W_c: store 1 / 2^(m_c - m*) now, times Z below
      reinterpret_cast<double*>(sC)[cskew(c0 + i)] = w > 0.0 ? 1.0 / (double)w32 : 0.0;
      part += w;
      if (w > 0.0) lastpos = c0 + i;
    }
  } else {  // long sequences in 64-key chunks: the smem loop
    float mloc = -INFINITY;
    for (int c = tid; c < nC; c += NT) {
      const float2 v = __ldcg(cs + c);
      sC[cskew(c)] = v;
      mloc = fmaxf(mloc, v.x);
    }
    const float mstar = block_max_f(mloc, sred_f);  // (its barrier also publishes sC)
    SANTA_TRACE(3);
    for (int c = c0; c < c1; ++c) {
      const float2 st = sC[cskew(c)];
      const float w32 = st.y > 0.f ? ex2(st.x - mstar) : 0.f;
      const double w = (double)w32 * (double)st.y;
      sF[cskew(c)] = w;
      part += w;
      if (w > 0.0) lastpos = c;
    }
    __syncthreads();  // every thread has read its sC entries before they are overwritten
    for (int c = c0; c < c1; ++c) {
      const double w = sF[cskew(c)];
      reinterpret_cast<double*>(sC)[cskew(c)] = w > 0.0 ? (double)sC[cskew(c)].y / w : 0.0;  // l_c / W_c
    }
  }
  double Z;
  double run = block_excl_scan_d(part, sred_d, &Z);
  lastpos = block_max_i(lastpos, sred_i);
  const double invZ = 1.0 / Z;
  for (int c = c0; c < c1; ++c) {
    const double w = sF[cskew(c)];
    run += w;
    sF[cskew(c)] = c >= lastpos ? 1.0 : run * invZ;
    reinterpret_cast<double*>(sC)[cskew(c)] *= Z;  // Z l_c / W_c
  }
  SANTA_TRACE(4);
  // ---- sequence sharding: this rank's slice of the global shard CDF --------------------------
  if (tid == 0) {
    sTlo = 0.0;
    sThi = 2.0;
    sTscale = 1.0;
    sOwnAny = 1;
    if (p.stats_all) {
      const size_t stride = (size_t)p.B * p.H * 2;
      double ms = -INFINITY;
      int lastr = 0;
      for (int r = 0; r < p.world; ++r) {
        ms = fmax(ms, p.stats_all[r * stride + bh * 2]);
        if (p.stats_all[r * stride + bh * 2 + 1] > 0.0) lastr = r;
      }
      double Zg = 0.0, Wr = 0.0, lo = 0.0, hi = 0.0, cum = 0.0;
      for (int r = 0; r < p.world; ++r) {
        const double Lr = p.stats_all[r * stride + bh * 2 + 1];
        const double W = Lr > 0.0 ? exp2(p.stats_all[r * stride + bh * 2] - ms) * Lr : 0.0;
        if (r == p.rank) Wr = W;
        Zg += W;
      }
      for (int r = 0; r <= p.rank; ++r) {
        const double Lr = p.stats_all[r * stride + bh * 2 + 1];
        const double W = Lr > 0.0 ? exp2(p.stats_all[r * stride + bh * 2] - ms) * Lr : 0.0;
        lo = cum / Zg;
        cum += W;
        hi = (r >= lastr) ? 1.0 : cum / Zg;
      }
      sTlo = lo;
      sThi = hi;
      sTscale = Zg / Wr;
      sOwnAny = Wr > 0.0 ? 1 : 0;
    }
  }
  __syncthreads();

  // ---- a5 (part 1): chunk of every sample (thread per sample, shared-memory search) ------------
  for (int m = tid; m < Sl; m += NT) {
    double Tm = sT[m];
    int c = -1;
    bool own = true;
    if (p.stats_all) {
      own = sOwnAny && Tm >= sTlo && Tm < sThi;
      Tm = (Tm - sTlo) * sTscale;
    }
    float tl = 0.f;
    if (own) {
      int lo = 0, hi = nC - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sF[cskew(mid)] > Tm) hi = mid; else lo = mid + 1;
      }
      c = lo;
      const double Fprev = c ? sF[cskew(c - 1)] : 0.0;
      tl = __double2float_rd((Tm - Fprev) * reinterpret_cast<const double*>(sC)[cskew(c)]);
    }
    sChunk[m] = c;
    sTl[m] = tl;
  }
  __syncthreads();
  SANTA_TRACE(5);

  // ---- a5 (part 2) + a6 ---------------------------------------------------------------------------
  if constexpr (UMAX <= 4)  // 4 prefix blocks, then 8 V rows in flight per half-warp: no spills at 64 registers
    gather_chunk_rows_2ph<T, D, false, 4, 8>(p, b, h, rank, kvh, bh, Sl, m_lo, seqlen, sChunk, sTl, sRed, sPart, nullptr,
                                          -1);
  else
    gather_chunk_rows<T, D>(p, b, h, rank, kvh, bh, Sl, m_lo, seqlen, sChunk, sTl, sRed, sPart);
  return sPart;
}

template <typename T, int D>
__device__ __forceinline__ void store_out(const SampleParams& p, size_t bh, int d, float v) {
  if (p.out_f32) p.out_f32[bh * D + d] = v;
  else reinterpret_cast<T*>(p.out)[bh * D + d] = Elem<T>::from_f(v);
}

// Sum the partials of the CS CTAs of one head's cluster (through DSMEM, fixed rank order), scale
// by 1/S and store the head's output.
template <typename T, int D>
__device__ __forceinline__ void finish_head(const SampleParams& p, size_t bh, int rank, int CS, float* sPart,
                                            float scale = -1.f) {
  namespace cg = cooperative_groups;
  const float invS = scale >= 0.f ? scale : 1.0f / (float)p.S;
  if (CS > 1) {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (rank == 0)
      for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float s = 0.f;
        for (int r = 0; r < CS; ++r) s += cluster.map_shared_rank(sPart, r)[d];
        store_out<T, D>(p, bh, d, s * invS);
      }
    cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
  } else {
    for (int d = threadIdx.x; d < D; d += blockDim.x) store_out<T, D>(p, bh, d, sPart[d] * invS);
  }
}

// MINB = resident CTAs per SM the registers are capped for: 1 (default, 8 samples in flight per
// half-warp, fused prefix-block -> V-row loop) or 4 (<= 64 registers, two-phase gather: 4 prefix
// blocks, then 8 V rows in flight per half-warp -- no spills; (8, 8) spilled 160 B and ran 5 us slower
// at config 5): large batches (config 5: 512 heads = 512 CTAs) fit in ONE wave at 4 CTAs per SM
// instead of two at 2 (config 5 175.6 -> 162.1 us).
template <typename T, int D, int G, int MINB = 1>
__global__ void __launch_bounds__(kSampleThreads, MINB) sample_gather_kernel(SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  namespace cg = cooperative_groups;
  const int CS = p.cluster;
  const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int h = blockIdx.x / CS, b = blockIdx.y;
  const size_t bh = (size_t)b * p.H + h;
  float* sPart = sample_item<T, D, G, (MINB >= 3 ? 4 : 8)>(p, b, h, rank, CS, smem_raw);
  finish_head<T, D>(p, bh, rank, CS, sPart);
  if (p.trace && threadIdx.x == 0 && rank == 0) p.trace[bh * 16 + 7] = gtimer();
}

}  // namespace santa
