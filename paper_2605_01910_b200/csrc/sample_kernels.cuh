// sample_kernels.cuh -- combine + sampler + gather-add of the SANTA decode hot path
// (SURVEY sec. 8(a) rows a3-a6).
//
// One CTA = one (batch, kv-head, split); it owns strata m in [m0, m1) of ALL G heads of
// the group.  Steps:
//  a3 combine: per head, m* = max_c m_c, W_c = 2^(m_c - m*) l_c, fp64 inclusive scan ->
//     chunk CDF F_c = sum_{c'<=c} W_c' / Z, clamped to 1 after the last positive chunk
//     (reading #5).  (Same LSE merge as Alg. prop-budgets P:1606-1607 / flash-k2 P:1701.)
//  a4 thresholds: Philox4x32-10, T_m in fp64 exactly as the oracle (reading #1-#3).
//  a5 inverse CDF: c = min{c : F_c > T}; then within the chunk the rescaled threshold
//     t = (T - F_{c-1}) Z 2^(m* - m_c) is compared (fp64) with the fp32 prefix stash:
//     k = min{k : P_c[k] > t}  (J = min{j : F(j) > T}, reading #4).
//  a6 gather-add: rows are read once per run of equal consecutive indices of a head
//     (stratified/systematic indices are non-decreasing in m) and added count times
//     (count * v is exact: small integer times a bf16 value), fp32 accumulators, 1/S and
//     the cast in the epilogue ("adds only", Table).
//  Cross-split reduction: each split writes its fp32 partial; the last CTA of the
//  (b, kv-head) (atomic ticket) sums the splits in a FIXED order -> deterministic output.
//
// Sequence-sharded mode (stats_all != NULL, reading #18): the global threshold T is first
// located in the shard CDF built from every rank's (m_r, L_r); strata outside this rank's
// [F_{r-1}, F_r) are skipped, owned ones are re-normalised to the local distribution.
#pragma once
#include "common.cuh"
#include "philox.cuh"

namespace santa {

constexpr int kSampleThreads = 256;

struct SampleParams {
  const float* stash;
  const float2* cstats;
  int Cmax, stash_stride;
  const void* V;
  KvLayout kv;
  const int32_t* seqlens;
  int B, H, Hkv, S, mode, nsplit, max_loc;
  uint64_t seed, offset;
  int batch_offset, head_offset;
  void* out;            // [B, H, D] dtype T (standard mode)
  float* out_f32;       // [B, H, D] fp32 (seq-shard partial mode) -- used if non-NULL
  int32_t* idx_out;     // [B, H, S] or NULL
  float* partial;       // [B*Hkv, nsplit, G, D]
  uint32_t* tickets;    // [B*Hkv]
  uint32_t* flags;
  // sequence sharding
  const double* stats_all;  // [world, B, H, 2] or NULL
  int rank, world;
  const int32_t* token_offset;  // [B] or NULL
};

// block-wide exclusive scan of one double per thread; returns exclusive prefix, sets *total
__device__ __forceinline__ double block_excl_scan_d(double v, double* sred, double* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double incl = warp_incl_scan_d(v, lane);
  if (lane == 31) sred[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double w = lane < kSampleThreads / 32 ? sred[lane] : 0.0;
    const double wi = warp_incl_scan_d(w, lane);
    if (lane < kSampleThreads / 32) sred[lane] = wi - w;
    if (lane == kSampleThreads / 32 - 1) sred[32] = wi;
  }
  __syncthreads();
  const double r = sred[warp] + incl - v;
  *total = sred[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ float block_max_f(float v, float* sredf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) sredf[warp] = v;
  __syncthreads();
  float r = sredf[0];
#pragma unroll
  for (int w = 1; w < kSampleThreads / 32; ++w) r = fmaxf(r, sredf[w]);
  __syncthreads();
  return r;
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kSampleThreads) sample_gather_kernel(SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sF = reinterpret_cast<double*>(smem_raw);               // [G][Cmax]
  int* sIdx = reinterpret_cast<int*>(sF + (size_t)G * p.Cmax);     // [G][max_loc]
  __shared__ double sred[33];
  __shared__ float sredf[8];
  __shared__ double sMstar[G], sZ[G], sTlo[G], sThi[G], sTscale[G];
  __shared__ int sOwnAny[G];
  __shared__ int sLast;

  pdl_wait_primary();

  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x;
  const int seqlen = __ldg(p.seqlens + b);
  const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
  const int m0 = (int)((int64_t)split * p.S / p.nsplit);
  const int m1 = (int)((int64_t)(split + 1) * p.S / p.nsplit);
  const int nloc = m1 - m0;

  if (seqlen < 1) {  // empty distribution: zero output, flag, no sampling
    if (split == 0) {
      for (int t = tid; t < G * D; t += kSampleThreads) {
        const size_t o = (bh0 + t / D) * D + t % D;
        if (p.out_f32) p.out_f32[o] = 0.f;
        else reinterpret_cast<T*>(p.out)[o] = Elem<T>::from_f(0.f);
      }
      if (tid == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    }
    if (p.idx_out)
      for (int t = tid; t < G * nloc; t += kSampleThreads)
        p.idx_out[(bh0 + t / nloc) * p.S + m0 + t % nloc] = -1;
    return;
  }
  const int nC = (seqlen + kChunk - 1) / kChunk;

  // ---- a3: chunk CDF per head (fp64) ----------------------------------------------------
  const int per = (nC + kSampleThreads - 1) / kSampleThreads;
  for (int g = 0; g < G; ++g) {
    const float2* cs = p.cstats + (bh0 + g) * p.Cmax;
    float mloc = -INFINITY;
    for (int c = tid; c < nC; c += kSampleThreads) mloc = fmaxf(mloc, __ldcg(&cs[c].x));
    const float mstar = block_max_f(mloc, sredf);
    const int c0 = tid * per;
    double part = 0.0;
    for (int c = c0; c < min(c0 + per, nC); ++c) {
      const float2 st = __ldcg(&cs[c]);
      part += st.y > 0.f ? exp2((double)st.x - (double)mstar) * (double)st.y : 0.0;
    }
    double Z;
    double run = block_excl_scan_d(part, sred, &Z);
    for (int c = c0; c < min(c0 + per, nC); ++c) {
      const float2 st = __ldcg(&cs[c]);
      run += st.y > 0.f ? exp2((double)st.x - (double)mstar) * (double)st.y : 0.0;
      sF[g * p.Cmax + c] = run / Z;
    }
    if (tid == 0) {
      sMstar[g] = (double)mstar;
      sZ[g] = Z;
    }
    __syncthreads();
    // clamp to 1 from the last positive-mass chunk on (reading #5)
    if (tid == 0) {
      int last = nC - 1;
      while (last > 0 && __ldcg(&cs[last].y) <= 0.f) --last;
      for (int c = last; c < nC; ++c) sF[g * p.Cmax + c] = 1.0;
    }
  }
  // ---- sequence sharding: this rank's slice of the global shard CDF ----------------------
  if (tid < G) {
    const int g = tid;
    sTlo[g] = 0.0;
    sThi[g] = 2.0;
    sTscale[g] = 1.0;
    sOwnAny[g] = 1;
    if (p.stats_all) {
      const size_t h = bh0 + g;
      const size_t stride = (size_t)p.B * p.H * 2;
      double ms = -INFINITY;
      for (int r = 0; r < p.world; ++r) ms = fmax(ms, p.stats_all[r * stride + h * 2]);
      double Zg = 0.0, lo = 0.0, Wr = 0.0;
      int lastpos = 0;
      for (int r = 0; r < p.world; ++r) {
        const double L = p.stats_all[r * stride + h * 2 + 1];
        if (L > 0.0) lastpos = r;
      }
      for (int r = 0; r < p.world; ++r) {
        const double L = p.stats_all[r * stride + h * 2 + 1];
        const double W = L > 0.0 ? exp2(p.stats_all[r * stride + h * 2] - ms) * L : 0.0;
        if (r == p.rank) Wr = W;
        Zg += W;
      }
      double cum = 0.0, hi = 0.0;
      for (int r = 0; r <= p.rank; ++r) {
        const double L = p.stats_all[r * stride + h * 2 + 1];
        const double W = L > 0.0 ? exp2(p.stats_all[r * stride + h * 2] - ms) * L : 0.0;
        lo = cum / Zg;
        cum += W;
        hi = (r >= lastpos) ? 1.0 : cum / Zg;
      }
      sTlo[g] = lo;
      sTscale[g] = Zg / Wr;
      sOwnAny[g] = (Wr > 0.0) ? 1 : 0;
      sThi[g] = hi;
    }
  }
  __syncthreads();

  // ---- a4 + a5: thresholds and inverse CDF ---------------------------------------------
  for (int t = tid; t < G * nloc; t += kSampleThreads) {
    const int g = t / nloc, m = m0 + t % nloc;
    const int h = kvh * G + g;
    PhiloxStream ps(p.seed, p.offset, kTagValueSampler, (uint32_t)(p.head_offset + h),
                    (uint32_t)(p.batch_offset + b));
    double T = sample_threshold(p.mode, m, p.S, ps);
    int j = -1;
    bool own = true;
    if (p.stats_all) {
      own = sOwnAny[g] && T >= sTlo[g] && T < sThi[g];
      T = (T - sTlo[g]) * sTscale[g];
    }
    if (own) {
      const double* F = sF + g * p.Cmax;
      int lo = 0, hi = nC - 1;  // c = min{c : F_c > T}
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (F[mid] > T) hi = mid; else lo = mid + 1;
      }
      const int c = lo;
      const double Fprev = c ? F[c - 1] : 0.0;
      const float2 st = __ldcg(&p.cstats[(bh0 + g) * p.Cmax + c]);
      const double tl = (T - Fprev) * sZ[g] * exp2(sMstar[g] - (double)st.x);
      const float* P = p.stash + (bh0 + g) * p.stash_stride + (size_t)c * kChunk;
      const int n = min(kChunk, seqlen - c * kChunk);
      int a = 0, e = n;  // k = min{k : P[k] > tl}
      while (a < e) {
        const int mid = (a + e) >> 1;
        if ((double)__ldcg(P + mid) > tl) e = mid; else a = mid + 1;
      }
      if (a >= n) {  // threshold beyond the chunk total (rounding): last positive-mass key
        const float tot = __ldcg(P + n - 1);
        a = 0; e = n - 1;
        while (a < e) {
          const int mid = (a + e) >> 1;
          if (__ldcg(P + mid) >= tot) e = mid; else a = mid + 1;
        }
      }
      j = c * kChunk + a;
    }
    sIdx[g * p.max_loc + (m - m0)] = j;
    if (p.idx_out)
      p.idx_out[(bh0 + g) * p.S + m] = (j >= 0 && p.token_offset) ? j + __ldg(p.token_offset + b) : j;
  }
  __syncthreads();

  // ---- a6: gather-add ------------------------------------------------------------------
  constexpr int EB = (int)sizeof(T);
  constexpr int RPG = D * EB / 16;          // lanes per V row (16 B each)
  constexpr int EPL = 16 / EB;              // elements per lane
  constexpr int NRG = kSampleThreads / RPG; // row groups per CTA
  static_assert(NRG >= G, "row groups");
  constexpr int GPH = NRG / G;              // row groups per head
  const int rg = tid / RPG, l = tid % RPG;
  float acc[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
  const int gh = rg % G, sub = rg / G;
  if (sub < GPH) {
    const int* idx = sIdx + gh * p.max_loc;
    const T* Vb = reinterpret_cast<const T*>(p.V);
    for (int i = sub; i < nloc; i += GPH) {
      const int j = idx[i];
      if (j < 0 || (i > 0 && idx[i - 1] == j)) continue;  // skipped / counted by the run head
      int cnt = 1;
      while (i + cnt < nloc && idx[i + cnt] == j) ++cnt;
      const uint4 raw = ldg_nc(Vb + p.kv.row(b, kvh, j, D) + l * EPL);
      const float fc = (float)cnt;
      if constexpr (EB == 2) {
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[2 * e] = fmaf(fc, Elem<T>::lo(w[e]), acc[2 * e]);
          acc[2 * e + 1] = fmaf(fc, Elem<T>::hi(w[e]), acc[2 * e + 1]);
        }
      } else {
        acc[0] = fmaf(fc, __uint_as_float(raw.x), acc[0]);
        acc[1] = fmaf(fc, __uint_as_float(raw.y), acc[1]);
        acc[2] = fmaf(fc, __uint_as_float(raw.z), acc[2]);
        acc[3] = fmaf(fc, __uint_as_float(raw.w), acc[3]);
      }
    }
  }
  // reduce row groups of the same head in a fixed order through shared memory
  float* sRed = reinterpret_cast<float*>(sIdx + G * p.max_loc);  // [NRG][RPG*EPL] = [NRG][D]
#pragma unroll
  for (int e = 0; e < EPL; ++e) sRed[rg * D + l * EPL + e] = acc[e];
  __syncthreads();
  float* part = p.partial + (((size_t)b * p.Hkv + kvh) * p.nsplit + split) * G * D;
  for (int t = tid; t < G * D; t += kSampleThreads) {
    const int g = t / D, d = t % D;
    float s = 0.f;
    for (int sb = 0; sb < GPH; ++sb) s += sRed[(sb * G + g) * D + d];
    part[t] = s;
  }
  // ---- cross-split deterministic reduction (last CTA) -----------------------------------
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const uint32_t prev = atomicAdd(p.tickets + (size_t)b * p.Hkv + kvh, 1u);
    sLast = (prev == (uint32_t)(p.nsplit - 1));
  }
  __syncthreads();
  if (!sLast) return;
  __threadfence();
  const float invS = 1.0f / (float)p.S;
  const float* part0 = p.partial + ((size_t)b * p.Hkv + kvh) * p.nsplit * G * D;
  for (int t = tid; t < G * D; t += kSampleThreads) {
    float s = 0.f;
    for (int sp = 0; sp < p.nsplit; ++sp) s += __ldcg(part0 + (size_t)sp * G * D + t);
    const size_t o = bh0 * D + t;
    if (p.out_f32) p.out_f32[o] = s * invS;
    else reinterpret_cast<T*>(p.out)[o] = Elem<T>::from_f(s * invS);
  }
  if (tid == 0) p.tickets[(size_t)b * p.Hkv + kvh] = 0u;
}

}  // namespace santa
