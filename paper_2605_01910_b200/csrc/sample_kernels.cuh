// sample_kernels.cuh -- combine + sampler + gather-add of the SANTA decode hot path
// (SURVEY sec. 8(a) rows a3-a6).
//
// One CTA = one (batch, query head): it owns all S strata of that head, so no cross-CTA
// reduction is needed and the chunk CDF is built exactly once per head.  Steps:
//  a4 thresholds (before griddepcontrol.wait, overlapping the score pass): Philox4x32-10,
//     T_m in fp64 exactly as the oracle (readings #1-#3).
//  a3 combine: the head's chunk stats are loaded in one round trip; m* = max_c m_c,
//     W_c = 2^(m_c - m*) l_c (fp64), block-wide fp64 scan -> F_c = sum_{c'<=c} W / Z, clamped
//     to 1 from the last positive chunk on (reading #5).  (The LSE merge of Alg.
//     prop-budgets P:1606-1607 / flash-k2 P:1701, in fp64.)
//  a5 inverse CDF: c = min{c : F_c > T} (binary search in shared memory), then the rescaled
//     threshold t = (T - F_{c-1}) Z 2^(m* - m_c) is located in the chunk's fp32 prefix stash by
//     a 16-ary search (2 dependent L2 round trips for L <= 256):
//     k = min{k : P_c[k] > t}; J = c L + k  (J = min{j : F(j) > T}, reading #4).
//  a6 gather-add: runs of equal consecutive indices (stratified/systematic indices are
//     non-decreasing in m) are read once and added `count` times (count * v is exact for a
//     small integer count and a bf16 v); 16 rows in flight per lane group; fp32 accumulators;
//     1/S and the cast in the epilogue ("adds only", Table).
//     V rows shared by the G heads of a group are deduplicated by the L2 (the G CTAs of a
//     group run concurrently), not in shared memory.
//
// Sequence-sharded mode (stats_all != NULL, reading #18): the global threshold T is first
// located in the shard CDF built from every rank's (m_r, L_r); strata outside this rank's
// [F_{r-1}, F_r) are skipped, owned ones are re-normalised to the local distribution.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "philox.cuh"

namespace santa {

constexpr int kSampleThreads = 256;
constexpr int kMaxBudget = 4096;   // S limit (shared-memory sample tables)

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
  void* out;            // [B, H, D] dtype T (standard mode)
  float* out_f32;       // [B, H, D] fp32 (seq-shard partial mode) -- used if non-NULL
  int32_t* idx_out;     // [B, H, S] or NULL
  uint32_t* flags;
  // sequence sharding
  const double* stats_all;  // [world, B, H, 2] or NULL
  int rank, world;
  const int32_t* token_offset;  // [B] or NULL
  int cluster;                  // CTAs per head (thread-block cluster size, 1..8)
  unsigned long long* trace;    // NULL in the library; tools/microbench_sample.cu phase timing
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SANTA_TRACE(i) \
  if (p.trace && threadIdx.x == 0 && (blockIdx.x % p.cluster) == 0) \
  p.trace[(blockIdx.y * gridDim.x + blockIdx.x) / p.cluster * 16 + (i)] = gtimer()

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

__device__ __forceinline__ float block_max_f(float v, float* sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  float r = sred[0];
#pragma unroll
  for (int w = 1; w < kSampleThreads / 32; ++w) r = fmaxf(r, sred[w]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ int block_max_i(int v, int* sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  int r = sred[0];
#pragma unroll
  for (int w = 1; w < kSampleThreads / 32; ++w) r = max(r, sred[w]);
  __syncthreads();
  return r;
}

// block-wide exclusive scan of one double per thread; *total receives the sum
__device__ __forceinline__ double block_excl_scan_d(double v, double* sred, double* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double incl = warp_incl_scan_d(v, lane);
  if (lane == 31) sred[warp] = incl;
  __syncthreads();
  double off = 0.0, tot = 0.0;
#pragma unroll
  for (int w = 0; w < kSampleThreads / 32; ++w) {
    const double x = sred[w];
    if (w < warp) off += x;
    tot += x;
  }
  __syncthreads();
  *total = tot;
  return off + incl - v;
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kSampleThreads, 1) sample_gather_kernel(SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sF = reinterpret_cast<double*>(smem_raw);               // [Cmax]
  double* sT = sF + p.Cmax;                                        // [S]  (reused: see sR)
  float2* sC = reinterpret_cast<float2*>(sT + p.S);                // [Cmax]
  int* sIdx = reinterpret_cast<int*>(sC + p.Cmax);                 // [S]
  int* sCnt = sIdx + p.S;                                          // [S]
  float* sRed = reinterpret_cast<float*>(sCnt + p.S);              // [NRG][D]
  __shared__ double sred_d[kSampleThreads / 32];
  __shared__ float sred_f[kSampleThreads / 32];
  __shared__ int sred_i[kSampleThreads / 32];
  __shared__ double sTlo, sThi, sTscale;
  __shared__ int sOwnAny;

  // grid.x = H * CS: the CS CTAs of head h form one thread-block cluster; CTA rank r owns the
  // strata [m_lo, m_hi) and the cluster sums the partial outputs through distributed shared memory.
  namespace cg = cooperative_groups;
  const int CS = p.cluster;
  const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int h = blockIdx.x / CS, b = blockIdx.y, kvh = h / G;
  const int tid = threadIdx.x;
  const size_t bh = (size_t)b * p.H + h;
  const int S = p.S;                                   // global budget (thresholds, 1/S)
  const int m_lo = (int)((long long)S * rank / CS), m_hi = (int)((long long)S * (rank + 1) / CS);
  const int Sl = m_hi - m_lo;                          // strata owned by this CTA

  SANTA_TRACE(0);
  // ---- a4: thresholds (independent of the score pass) ---------------------------------------
  {
    PhiloxStream ps(p.seed, p.offset, kTagValueSampler, (uint32_t)(p.head_offset + h), (uint32_t)(p.batch_offset + b));
    for (int i = tid; i < Sl; i += kSampleThreads) sT[i] = sample_threshold(p.mode, m_lo + i, S, ps);
  }

  SANTA_TRACE(1);
  pdl_wait_primary();
  SANTA_TRACE(2);

  const int seqlen = __ldg(p.seqlens + b);
  if (seqlen < 1) {  // empty distribution: zero output, flag, no sampling (cluster-uniform)
    if (rank == 0) {
      for (int d = tid; d < D; d += kSampleThreads) {
        if (p.out_f32) p.out_f32[bh * D + d] = 0.f;
        else reinterpret_cast<T*>(p.out)[bh * D + d] = Elem<T>::from_f(0.f);
      }
      if (tid == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    }
    if (p.idx_out)
      for (int i = tid; i < Sl; i += kSampleThreads) p.idx_out[bh * S + m_lo + i] = -1;
    return;
  }
  const int nC = (seqlen + p.L - 1) / p.L;

  // ---- a3: chunk stats -> fp64 chunk CDF ------------------------------------------------------
  const float2* cs = p.cstats + bh * p.Cmax;
  float mloc = -INFINITY;
  for (int c = tid; c < nC; c += kSampleThreads) {
    const float2 v = __ldcg(cs + c);
    sC[c] = v;
    mloc = fmaxf(mloc, v.x);
  }
  const float mstar = block_max_f(mloc, sred_f);  // (its barrier also publishes sC)
  SANTA_TRACE(3);
  const int per = (nC + kSampleThreads - 1) / kSampleThreads;
  const int c0 = tid * per, c1 = min(c0 + per, nC);
  double part = 0.0;
  int lastpos = -1;
  for (int c = c0; c < c1; ++c) {
    const float2 st = sC[c];
    const double w = st.y > 0.f ? exp2((double)st.x - (double)mstar) * (double)st.y : 0.0;
    sF[c] = w;
    part += w;
    if (w > 0.0) lastpos = c;
  }
  double Z;
  double run = block_excl_scan_d(part, sred_d, &Z);
  lastpos = block_max_i(lastpos, sred_i);
  const double invZ = 1.0 / Z;
  for (int c = c0; c < c1; ++c) {
    const double w = sF[c];
    run += w;
    sF[c] = c >= lastpos ? 1.0 : run * invZ;
    // rescale factor of the in-chunk search, Z * 2^(m* - m_c) = Z l_c / W_c, kept in the
    // (now unused) float2 slot of the chunk as a double
    reinterpret_cast<double*>(sC)[c] = w > 0.0 ? Z * (double)sC[c].y / w : 0.0;
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
  // c = min{c : F_c > T}; the in-chunk threshold t = (T - F_{c-1}) Z 2^(m* - m_c) is kept as
  // rd(t) (fp32, rounded toward -inf), which decides P[k] > t exactly (see chunk_count).
  int* sChunk = reinterpret_cast<int*>(sCnt);        // [S] chunk of sample m (-1: not owned)
  float* sTl = reinterpret_cast<float*>(sIdx);       // [S] rd(t)
  for (int m = tid; m < Sl; m += kSampleThreads) {
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
        if (sF[mid] > Tm) hi = mid; else lo = mid + 1;
      }
      c = lo;
      const double Fprev = c ? sF[c - 1] : 0.0;
      tl = __double2float_rd((Tm - Fprev) * reinterpret_cast<const double*>(sC)[c]);
    }
    sChunk[m] = c;
    sTl[m] = tl;
  }
  __syncthreads();
  SANTA_TRACE(5);

  // ---- a5 (part 2) + a6: half-warp per sample: in-chunk search + gather-add ---------------------
  // 16 lanes load the sample's chunk prefix block coalesced (one 16-B load each for L = 64),
  // count P[k] <= rd(t) with ballots (= min{k : P[k] > t}), then the same 16 lanes load the V
  // row (16 B each) and add it.  U samples are in flight per half-warp (2 dependent L2/DRAM
  // round trips for the whole budget when S <= 16 * U * 16).
  constexpr int EB = (int)sizeof(T);
  constexpr int VCH = D * EB / 16;                  // 16-B chunks per V row
  constexpr int NCH = (VCH + 15) / 16;              // chunks per lane
  constexpr int EPC = 16 / EB;                      // elements per chunk
  constexpr int NHW = kSampleThreads / 16;          // half-warps
  constexpr int U = 8;
  const int hw = tid >> 4, l = tid & 15;
  const unsigned hmask = 0xffffu << (threadIdx.x & 16);
  float acc[NCH][EPC];
#pragma unroll
  for (int q = 0; q < NCH; ++q)
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[q][e] = 0.f;
  const T* Vb = reinterpret_cast<const T*>(p.V);
  const float* Pbase = p.stash + bh * p.stash_stride;
  const int tok0 = p.token_offset ? __ldg(p.token_offset + b) : 0;
  // warp-uniform trip count: warp w walks sample pairs 2w, 2w+1 (+ NHW per u); the full-mask
  // ballots below must be reached by both half-warps
  for (int mw = 2 * (tid >> 5); mw < Sl; mw += NHW * U) {
    const int m0 = mw + (hw & 1);
    int jj[U];
    // in-chunk search for U samples (loads first, then ballots)
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
      // warp-uniform: both half-warps execute every ballot with the full mask; inactive samples
      // have pv = +inf and tf = -inf, i.e. count 0
      const int m = m0 + u * NHW;
      const float tf = (cc[u] >= 0) ? sTl[m] : -INFINITY;
      const float4 v = pv[u];
      int k = __popc(__ballot_sync(0xffffffffu, v.x <= tf) & hmask) +
              __popc(__ballot_sync(0xffffffffu, v.y <= tf) & hmask) +
              __popc(__ballot_sync(0xffffffffu, v.z <= tf) & hmask) +
              __popc(__ballot_sync(0xffffffffu, v.w <= tf) & hmask);
      jj[u] = -1;
      if (cc[u] >= 0) {
        const float* P = Pbase + (size_t)cc[u] * p.L;
        if (p.L != 64) k = thread_chunk_search(P, nn[u], tf);
        if (k >= nn[u]) {  // rounding: threshold at/after the chunk total -> the last positive-mass key
          const float tot = __ldcg(P + nn[u] - 1);
          k = thread_chunk_search(P, nn[u], nextafterf(tot, -INFINITY));
        }
        jj[u] = cc[u] * p.L + k;
        if (l == 0 && p.idx_out) p.idx_out[bh * S + m_lo + m] = jj[u] + tok0;
      } else if (m < Sl && l == 0 && p.idx_out) {
        p.idx_out[bh * S + m_lo + m] = -1;  // stratum owned by another sequence shard
      }
    }
    // gather-add of the U rows
    uint4 raw[U][NCH];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        const int ch = l + 16 * q;
        raw[u][q] = (jj[u] >= 0 && ch < VCH) ? ldg_nc(Vb + p.kv.row(b, kvh, jj[u], D) + ch * EPC)
                                             : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        if constexpr (EB == 2) {
          const uint32_t w[4] = {raw[u][q].x, raw[u][q].y, raw[u][q].z, raw[u][q].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[q][2 * e] += Elem<T>::lo(w[e]);
            acc[q][2 * e + 1] += Elem<T>::hi(w[e]);
          }
        } else {
          acc[q][0] += __uint_as_float(raw[u][q].x);
          acc[q][1] += __uint_as_float(raw[u][q].y);
          acc[q][2] += __uint_as_float(raw[u][q].z);
          acc[q][3] += __uint_as_float(raw[u][q].w);
        }
      }
  }
  // deterministic reduction over the half-warps (fixed order), then over the cluster (fixed rank
  // order, through distributed shared memory)
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    const int ch = l + 16 * q;
    if (ch < VCH)
#pragma unroll
      for (int e = 0; e < EPC; ++e) sRed[hw * D + ch * EPC + e] = acc[q][e];
  }
  __syncthreads();
  SANTA_TRACE(6);
  float* sPart = sRed + NHW * D;  // [D] this CTA's partial sum
  for (int d = tid; d < D; d += kSampleThreads) {
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < NHW; ++r) s += sRed[r * D + d];
    sPart[d] = s;
  }
  const float invS = 1.0f / (float)S;
  if (CS > 1) {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // partials visible cluster-wide
    if (rank == 0) {
      for (int d = tid; d < D; d += kSampleThreads) {
        float s = 0.f;
        for (int r = 0; r < CS; ++r) s += cluster.map_shared_rank(sPart, r)[d];
        if (p.out_f32) p.out_f32[bh * D + d] = s * invS;
        else reinterpret_cast<T*>(p.out)[bh * D + d] = Elem<T>::from_f(s * invS);
      }
    }
    cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
  } else {
    __syncthreads();
    for (int d = tid; d < D; d += kSampleThreads) {
      if (p.out_f32) p.out_f32[bh * D + d] = sPart[d] * invS;
      else reinterpret_cast<T*>(p.out)[bh * D + d] = Elem<T>::from_f(sPart[d] * invS);
    }
  }
  SANTA_TRACE(7);
}

}  // namespace santa
