// score_kernels.cuh -- split-KV score pass of the SANTA decode hot path (SURVEY sec. 8(a)
// rows a1-a2; PAPER Alg. prop-pass1 P:1577-1595 is the prior art).
//
// One CTA = one chunk of L = 256 keys of one (batch, kv-head); it scores the chunk for all
// G query heads of the GQA group, keeps the fp32 scores in shared memory, then writes
//   * chunk statistics (m_c = max_k s_k, l_c = sum_k 2^(s_k - m_c))   [B, H, C] float2
//   * the inclusive prefix P_c[k] = sum_{k'<=k} 2^(s_k' - m_c)       [B, H, C*L] fp32 stash
// with s in log2 units (scale * log2(e) folded in).  The stash is the paper's "score stash"
// ("negligible bandwidth (1/d_k)"); storing the PREFIX instead of u makes the
// inverse-CDF a plain binary search.
//
// Score math (bf16/fp16): [16 keys x d] . [d x G heads] is a dense contraction done with
// mma.sync.m16n8k16 (keys = M, heads = N padded to 8, d = K).  The A fragments are loaded
// straight from global memory with 128-bit loads: the contraction index d may be permuted
// freely as long as A (K rows) and B (q) use the same permutation, so each thread loads
// 16 contiguous bytes per (row, jj) and the warp's load instruction covers 8 rows x 64
// contiguous bytes (fully used 32-B sectors).  Permutation, for k-step ks = 2*jj + s and
// fragment column kc (tig = lane & 3):
//   kc in {2tig, 2tig+1}   <-> d = 8*(4jj+tig) + 4s + (kc & 1)        (word 2s of the chunk)
//   kc in {2tig+8, 2tig+9} <-> d = 8*(4jj+tig) + 4s + 2 + (kc & 1)    (word 2s+1)
// It does not depend on the row (groupID), as the MMA requires.
#pragma once
#include "common.cuh"

namespace santa {

struct ScoreParams {
  const void* q;            // [B, H, D]
  const void* K;            // layout per kv
  KvLayout kv;
  const int32_t* seqlens;   // [B]
  int B, H, Hkv;
  float scale_log2;         // scale * log2(e)
  float* stash;             // [B, H, stash_stride] or NULL
  float2* cstats;           // [B, H, Cmax]
  int Cmax;
  int stash_stride;         // Cmax * kChunk
  uint32_t* tickets;        // [B * Hkv], zeroed here for the sample kernel
  uint32_t* flags;          // zeroed here (CTA 0,0,0)
};

// Scores of chunk keys [chunk_start, chunk_start + 256) (valid: first n_valid) for the G heads
// of kv-head kvh, written to sS[g * 256 + k] in log2 units; masked keys get -inf.
template <typename T, int D, int G>
__device__ __forceinline__ void score_chunk_mma(const T* __restrict__ qg /* q + (b*H + kvh*G)*D */,
                                                const T* __restrict__ K, const KvLayout& kv, int b,
                                                int kvh, int chunk_start, int n_valid,
                                                float scale_log2, float* sS) {
  static_assert(D == 64 || D == 128, "head_dim");
  static_assert(G >= 1 && G <= 8, "group size");
  constexpr int NJ = D / 32;           // 16-byte chunks per (thread, row)
  constexpr int TPW = kChunk / 16 / 4; // tiles per warp (4 warps)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;

  uint32_t qf[NJ][4];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    if (g < G) {
      const uint4 v = *reinterpret_cast<const uint4*>(qg + g * D + 8 * (4 * jj + tig));
      qf[jj][0] = v.x; qf[jj][1] = v.y; qf[jj][2] = v.z; qf[jj][3] = v.w;
    } else {
      qf[jj][0] = qf[jj][1] = qf[jj][2] = qf[jj][3] = 0u;
    }
  }

  uint4 kr[TPW][2][NJ];
#pragma unroll
  for (int i = 0; i < TPW; ++i) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int kl = 64 * warp + 16 * i + g + 8 * r;  // key index within the chunk
      if (kl < n_valid) {
        const T* row = K + kv.row(b, kvh, chunk_start + kl, D);
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) kr[i][r][jj] = ldg_stream(row + 8 * (4 * jj + tig));
      } else {
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) kr[i][r][jj] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
  }

#pragma unroll
  for (int i = 0; i < TPW; ++i) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
      Mma<T>::run(acc, kr[i][0][jj].x, kr[i][1][jj].x, kr[i][0][jj].y, kr[i][1][jj].y, qf[jj][0], qf[jj][1]);
      Mma<T>::run(acc, kr[i][0][jj].z, kr[i][1][jj].z, kr[i][0][jj].w, kr[i][1][jj].w, qf[jj][2], qf[jj][3]);
    }
    const int k0 = 64 * warp + 16 * i + g, k1 = k0 + 8;
    const int h0 = 2 * tig;
    if (h0 < G) {
      sS[h0 * kChunk + k0] = k0 < n_valid ? acc[0] * scale_log2 : -INFINITY;
      sS[h0 * kChunk + k1] = k1 < n_valid ? acc[2] * scale_log2 : -INFINITY;
    }
    if (h0 + 1 < G) {
      sS[(h0 + 1) * kChunk + k0] = k0 < n_valid ? acc[1] * scale_log2 : -INFINITY;
      sS[(h0 + 1) * kChunk + k1] = k1 < n_valid ? acc[3] * scale_log2 : -INFINITY;
    }
  }
}

// fp32 path (config C1 and any fp32 cache): plain FMA dot products, LPR lanes per key row.
template <int D, int G>
__device__ __forceinline__ void score_chunk_simt(const float* __restrict__ qg, const float* __restrict__ K,
                                                 const KvLayout& kv, int b, int kvh, int chunk_start,
                                                 int n_valid, float scale_log2, float* sS) {
  constexpr int LPR = D / 4;          // lanes per row (16 B each)
  constexpr int RPW = 32 / LPR;       // rows per warp step
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, l = lane % LPR;
  float qv[G][4];
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    const float4 v = *reinterpret_cast<const float4*>(qg + gg * D + 4 * l);
    qv[gg][0] = v.x; qv[gg][1] = v.y; qv[gg][2] = v.z; qv[gg][3] = v.w;
  }
  for (int k = 4 * 0 + warp * RPW + sub; k < kChunk; k += 4 * RPW) {
    float acc[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) acc[gg] = 0.f;
    if (k < n_valid) {
      const float4 v = *reinterpret_cast<const float4*>(K + kv.row(b, kvh, chunk_start + k, D) + 4 * l);
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
        acc[gg] = fmaf(qv[gg][0], v.x, fmaf(qv[gg][1], v.y, fmaf(qv[gg][2], v.z, qv[gg][3] * v.w)));
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) acc[gg] += __shfl_xor_sync(0xffffffffu, acc[gg], o);
      if (l == 0) sS[gg * kChunk + k] = k < n_valid ? acc[gg] * scale_log2 : -INFINITY;
    }
  }
}

// Per-head chunk max, exp2, inclusive prefix (stash) and (m_c, l_c).  Warp w handles heads
// w, w+4; lane handles 8 consecutive keys.  Requires __syncthreads() before the call.
template <int G>
__device__ __forceinline__ void chunk_stats_prefix(const float* sS, float* stash_h0, int stash_stride,
                                                   float2* cstats_h0, int Cmax) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int h = warp; h < G; h += 4) {
    const float4 a = *reinterpret_cast<const float4*>(sS + h * kChunk + 8 * lane);
    const float4 c = *reinterpret_cast<const float4*>(sS + h * kChunk + 8 * lane + 4);
    float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    float m = v[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) m = fmaxf(m, v[e]);
    m = warp_max(m);
    const float ms = (m == -INFINITY) ? 0.f : m;
    float run = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      run += ex2(v[e] - ms);
      v[e] = run;
    }
    const float incl = warp_incl_scan(run, lane);
    const float excl = incl - run;
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] += excl;
    if (stash_h0) {
      float* dst = stash_h0 + (size_t)h * stash_stride + 8 * lane;
      *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (lane == 31) cstats_h0[(size_t)h * Cmax] = make_float2(m, v[7]);
  }
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kScoreThreads, 3) score_stats_kernel(ScoreParams p) {
  __shared__ __align__(16) float sS[G * kChunk];
  pdl_launch_dependents();
  const int c = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  if (c == 0 && threadIdx.x == 0) {
    if (p.tickets) p.tickets[b * p.Hkv + kvh] = 0u;
    if (b == 0 && kvh == 0 && p.flags) *p.flags = 0u;
  }
  const int seqlen = __ldg(p.seqlens + b);
  const int chunk_start = c * kChunk;
  const int n_valid = min(kChunk, seqlen - chunk_start);
  const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
  float2* cst = p.cstats + bh0 * p.Cmax + c;
  if (n_valid <= 0) {  // chunk past the end of this sequence (or empty sequence): zero mass
    if (threadIdx.x < G) cst[(size_t)threadIdx.x * p.Cmax] = make_float2(-INFINITY, 0.f);
    return;
  }
  if constexpr (sizeof(T) == 2) {
    score_chunk_mma<T, D, G>(reinterpret_cast<const T*>(p.q) + bh0 * D, reinterpret_cast<const T*>(p.K),
                             p.kv, b, kvh, chunk_start, n_valid, p.scale_log2, sS);
  } else {
    score_chunk_simt<D, G>(reinterpret_cast<const float*>(p.q) + bh0 * D,
                           reinterpret_cast<const float*>(p.K), p.kv, b, kvh, chunk_start, n_valid,
                           p.scale_log2, sS);
  }
  __syncthreads();
  chunk_stats_prefix<G>(sS, p.stash ? p.stash + bh0 * p.stash_stride + chunk_start : nullptr,
                        p.stash_stride, cst, p.Cmax);
}

}  // namespace santa
