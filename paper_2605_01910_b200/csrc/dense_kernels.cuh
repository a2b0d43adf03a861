// dense_kernels.cuh -- in-repo exact dense decode attention (the reference the SANTA
// latency is reported against): split-KV "flash-decoding" over the same chunks
// and the same score pass as the SANTA path, then an LSE combine (the merge of Alg.
// flash-k2, with exact weights).
//   partial kernel: per (chunk, kv-head, batch): s (mma.sync), m_c, u = 2^(s - m_c),
//                   l_c = sum u, o_c[g] = sum_k u_k V_k (fp32, CUDA-core FMA over V)
//   combine kernel: per (head, batch): m* = max m_c, O = sum 2^(m_c-m*) o_c / sum 2^(m_c-m*) l_c
#pragma once
#include "common.cuh"
#include "score_kernels.cuh"

namespace santa {

struct DenseParams {
  const void* q;
  const void* K;
  const void* V;
  KvLayout kv;
  const int32_t* seqlens;
  int B, H, Hkv;
  float scale_log2;
  float2* cstats;   // [B, H, Cmax]
  float* opart;     // [B, H, Cmax, D]
  int Cmax;
  void* out;
  uint32_t* flags;
};

template <typename T, int D, int G>
__global__ void __launch_bounds__(kScoreThreads, 3) dense_partial_kernel(DenseParams p) {
  __shared__ __align__(16) float sS[G * kDenseChunk];
  __shared__ __align__(16) float sO[4][G][D];
  pdl_launch_dependents();
  const int c = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  if (c == 0 && b == 0 && kvh == 0 && threadIdx.x == 0 && p.flags) *p.flags = 0u;
  const int seqlen = __ldg(p.seqlens + b);
  const int chunk_start = c * kDenseChunk;
  const int n_valid = min(kDenseChunk, seqlen - chunk_start);
  const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
  float2* cst = p.cstats + bh0 * p.Cmax + c;
  if (n_valid <= 0) {
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per-head max and u = 2^(s - m_c) in place; l_c
  for (int h = warp; h < G; h += 4) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = sS[h * kDenseChunk + 8 * lane + e];
    float m = v[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) m = fmaxf(m, v[e]);
    m = warp_max(m);
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[e] = ex2(v[e] - m);
      sum += v[e];
      sS[h * kDenseChunk + 8 * lane + e] = v[e];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) cst[(size_t)h * p.Cmax] = make_float2(m, sum);
  }
  __syncthreads();
  // o_c[g][:] = sum_k u[g][k] V[k][:]; warp w takes keys [64w, 64w+64); lane owns D/32 elements
  constexpr int EPL = D / 32;
  float acc[G][EPL];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[g][e] = 0.f;
  const T* Vb = reinterpret_cast<const T*>(p.V);
  constexpr int U = 8;
  for (int k0 = 64 * warp; k0 < 64 * warp + 64; k0 += U) {
    float vv[U][EPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u;
      if (k < n_valid) {
        const T* row = Vb + p.kv.row(b, kvh, chunk_start + k, D) + lane * EPL;
        if constexpr (sizeof(T) == 2) {
          if constexpr (EPL == 4) {
            const uint2 w = *reinterpret_cast<const uint2*>(row);
            vv[u][0] = Elem<T>::lo(w.x); vv[u][1] = Elem<T>::hi(w.x);
            vv[u][2] = Elem<T>::lo(w.y); vv[u][3] = Elem<T>::hi(w.y);
          } else {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(row);
            vv[u][0] = Elem<T>::lo(w); vv[u][1] = Elem<T>::hi(w);
          }
        } else {
#pragma unroll
          for (int e = 0; e < EPL; ++e) vv[u][e] = reinterpret_cast<const float*>(row)[e];
        }
      } else {
#pragma unroll
        for (int e = 0; e < EPL; ++e) vv[u][e] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float w = sS[g * kDenseChunk + k0 + u];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[g][e] = fmaf(w, vv[u][e], acc[g][e]);
      }
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < EPL; ++e) sO[warp][g][lane * EPL + e] = acc[g][e];
  __syncthreads();
  for (int t = threadIdx.x; t < G * D; t += kScoreThreads) {
    const int g = t / D, d = t % D;
    const float s = sO[0][g][d] + sO[1][g][d] + sO[2][g][d] + sO[3][g][d];
    p.opart[((bh0 + g) * p.Cmax + c) * D + d] = s;
  }
}

// LSE combine of the chunk partials, 256 threads per (b, h): chunk weights 2^(m_c - m*) in
// parallel, then each (d, quarter) thread sums a quarter of the chunks (8 loads in flight),
// quarters summed in fixed order.
template <typename T, int D>
__global__ void __launch_bounds__(256) dense_combine_kernel(DenseParams p) {
  __shared__ float sW[4096];  // max_seqlen <= 2^20 -> <= 4096 chunks
  __shared__ float sred[8];
  __shared__ float sAcc[256];
  pdl_wait_primary();
  const int h = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int seqlen = __ldg(p.seqlens + b);
  const size_t bh = (size_t)b * p.H + h;
  T* out = reinterpret_cast<T*>(p.out) + bh * D;
  if (seqlen < 1) {
    for (int d = tid; d < D; d += 256) out[d] = Elem<T>::from_f(0.f);
    if (tid == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    return;
  }
  const int nC = (seqlen + kDenseChunk - 1) / kDenseChunk;
  const float2* cs = p.cstats + bh * p.Cmax;
  float ms = -INFINITY;
  for (int c = tid; c < nC; c += 256) ms = fmaxf(ms, __ldcg(&cs[c].x));
  ms = warp_max(ms);
  if ((tid & 31) == 0) sred[tid >> 5] = ms;
  __syncthreads();
  ms = sred[0];
  for (int w = 1; w < 8; ++w) ms = fmaxf(ms, sred[w]);
  float den = 0.f;
  for (int c = tid; c < nC; c += 256) {
    const float2 st = __ldcg(&cs[c]);
    const float w = st.y > 0.f ? ex2(st.x - ms) : 0.f;
    sW[c] = w;
    den = fmaf(w, st.y, den);
  }
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  __shared__ float sden[8];
  if ((tid & 31) == 0) sden[tid >> 5] = den;
  const int d = tid % D, part = tid / D, nparts = 256 / D;
  float num = 0.f;
  for (int c0 = part * 8; c0 < nC; c0 += nparts * 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (c0 + u < nC) ? __ldcg(p.opart + (bh * p.Cmax + c0 + u) * D + d) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (c0 + u < nC) num = fmaf(sW[c0 + u], v[u], num);
  }
  sAcc[tid] = num;
  __syncthreads();
  if (tid < D) {
    float s = 0.f, dn = 0.f;
    for (int q = 0; q < nparts; ++q) s += sAcc[q * D + tid];
    for (int w = 0; w < 8; ++w) dn += sden[w];
    out[tid] = Elem<T>::from_f(s / dn);
  }
}

}  // namespace santa
