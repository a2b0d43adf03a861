// flash_kernels.cuh -- S^2ANTA-flash: uniform per-tile budgets + deferred LSE merge (SURVEY 8(f)
// NEXT-1; App. N: Kernel 1 P:1669-1689, Kernel 2 P:1691-1706).
//
// The estimator: T = ceil(n / B_tile) tiles, S_tile = max(1, round(S / T)) samples in EVERY tile
// (reading #26), drawn by systematic sampling inside the tile as if it held all the mass
// (invdelta = S_tile / l_t, offset a0_t = Philox tag 5, draw t), O~_t = sum of its rows, and the
// merge O = (1/Z) sum_t W_t O~_t / S_tile with W_t = exp(m_t - m*) l_t.
//
// B200 layout: the score pass (its L = 64-key chunk stats and prefix stash) is the tile pass; a
// flash tile is CPT = B_tile / L consecutive chunks, whose stats are merged on the fly
// (m_t = max m_c, l_t = sum 2^(m_c - m_t) l_c, in-tile prefix U = C_{c-1} + 2^(m_c - m_t) P_c[k]).
// One kernel per (b, h) cluster (PDL-chained) then draws every tile's S_tile rows -- the j-th row
// of tile t is min{n : U_n >= (j - a0_t) l_t / S_tile} (as in prop, reading #25) -- and gathers
// them with per-sample merge weights W_t / (Z S_tile) in fp32, so Kernel 2's merge is folded into
// the gather (no O~ partials in HBM).
#pragma once
#include "sample_kernels.cuh"

namespace santa {

// S_tile = max(1, floor(S / T + 1/2)) in integers
__host__ __device__ inline int flash_tile_budget(int T, int S) {
  const int st = (int)((2LL * S + T) / (2LL * T));
  return st > 0 ? st : 1;
}

__host__ __device__ inline size_t flash_smem_bytes(int Cmax, int CPT, int M_local, int D, int nthreads) {
  const size_t Tmax = (Cmax + CPT - 1) / CPT;
  return (size_t)Cmax * 16 + Tmax * 20 + (size_t)M_local * 12 + (size_t)(nthreads / 16 + 1) * D * 4 + 64;
}

template <typename T, int D, int G>
__device__ float* flash_item(const SampleParams& p, int b, int h, int rank, int CS, int CPT, int Mmax,
                             unsigned char* smem_raw) {
  const int NT = blockDim.x, NHW = NT >> 4;
  const int kvh = h / G;
  const int tid = threadIdx.x;
  const size_t bh = (size_t)b * p.H + h;
  const int Slmax = (Mmax + CS - 1) / CS;
  const int Tmax = (p.Cmax + CPT - 1) / CPT;
  double* sCum = reinterpret_cast<double*>(smem_raw);    // [Cmax] in-tile inclusive chunk masses
  double* sTL = sCum + p.Cmax;                           // [Tmax] l_t
  float2* sCs = reinterpret_cast<float2*>(sTL + Tmax);   // [Cmax] chunk stats
  float* sTM = reinterpret_cast<float*>(sCs + p.Cmax);   // [Tmax] m_t
  float* sTW = sTM + Tmax;                               // [Tmax] W_t / (Z S_tile)
  int* sTLast = reinterpret_cast<int*>(sTW + Tmax);      // [Tmax] last chunk of positive mass
  int* sChunk = sTLast + Tmax;                           // [Slmax]
  float* sTl = reinterpret_cast<float*>(sChunk + Slmax); // [Slmax]
  float* sWt = sTl + Slmax;                              // [Slmax] merge weights
  float* sRed = sWt + Slmax;                             // [NHW][D]
  float* sPart = sRed + NHW * D;                         // [D]
  __shared__ double sred_d[32];
  __shared__ float sred_f[32];

  pdl_wait_primary();
  pdl_launch_dependents();  // the next step's PDL-launched score pass may set up meanwhile
  const int seqlen = __ldg(p.seqlens + b);
  const int nC = seqlen > 0 ? (seqlen + p.L - 1) / p.L : 0;
  const int Tt = (nC + CPT - 1) / CPT;
  const int S_tile = seqlen > 0 ? flash_tile_budget(Tt, p.S) : 0;
  const int M = S_tile * Tt;  // rows drawn for this head
  const int m_lo = (int)((long long)M * rank / CS), m_hi = (int)((long long)M * (rank + 1) / CS);
  const int Sl = m_hi - m_lo;
  if (p.idx_out) {  // rows past this head's M (shorter sequences) read -1
    const int f_lo = (int)((long long)Mmax * rank / CS), f_hi = (int)((long long)Mmax * (rank + 1) / CS);
    for (int i = max(f_lo, M) + tid; i < f_hi; i += NT) p.idx_out[bh * Mmax + i] = -1;
    if (seqlen < 1)
      for (int i = f_lo + tid; i < min(f_hi, M); i += NT) p.idx_out[bh * Mmax + i] = -1;
  }
  if (seqlen < 1) {  // empty distribution: zero output, flag, no sampling
    for (int d = tid; d < D; d += NT) sPart[d] = 0.f;
    if (rank == 0 && tid == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    __syncthreads();
    return sPart;
  }

  // ---- chunk stats, m*, Z = sum_c 2^(m_c - m*) l_c (= sum_t W_t) ------------------------------
  const float2* cs = p.cstats + bh * p.Cmax;
  float mloc = -INFINITY;
  for (int c = tid; c < nC; c += NT) {
    const float2 v = __ldcg(cs + c);
    sCs[c] = v;
    mloc = fmaxf(mloc, v.x);
  }
  const float mstar = block_max_f(mloc, sred_f);
  const int per = (nC + NT - 1) / NT;
  const int c0 = min(tid * per, nC), c1 = min(c0 + per, nC);
  double part = 0.0;
  for (int c = c0; c < c1; ++c) {
    const float2 st = sCs[c];
    part += st.y > 0.f ? exp2((double)st.x - (double)mstar) * (double)st.y : 0.0;
  }
  double Z;
  (void)block_excl_scan_d(part, sred_d, &Z);

  // ---- tile stats once per tile: m_t, in-tile cumulative chunk masses, l_t, merge weight ---------
  {
    const double inv_ZS = 1.0 / (Z * (double)S_tile);
    for (int t = tid; t < Tt; t += NT) {
      const int cA = t * CPT, cB = min(cA + CPT, nC);
      float mt = -INFINITY;
      for (int c = cA; c < cB; ++c) mt = fmaxf(mt, sCs[c].x);
      double run = 0.0;
      int last = cA;
      for (int c = cA; c < cB; ++c) {
        const double e = exp2((double)sCs[c].x - (double)mt) * (double)sCs[c].y;
        run += e;
        sCum[c] = run;
        if (e > 0.0) last = c;
      }
      sTM[t] = mt;
      sTL[t] = run;
      sTLast[t] = last;
      sTW[t] = (float)(exp2((double)mt - (double)mstar) * run * inv_ZS);
    }
  }
  __syncthreads();

  // ---- every sample: tile, chunk inside the tile, in-chunk threshold, merge weight --------------
  {
    PhiloxStream ps(p.seed, p.offset, kTagFlashTileOffset, (uint32_t)(p.head_offset + h),
                    (uint32_t)(p.batch_offset + b));
    for (int i = tid; i < Sl; i += NT) {
      const int m = m_lo + i;
      const int t = m / S_tile;
      const int j = m - t * S_tile + 1;
      const int cA = t * CPT, last = sTLast[t];
      const double a0 = ps.uniform((uint32_t)t);
      const double tau = ((double)j - a0) * sTL[t] / (double)S_tile;
      // first chunk whose cumulative in-tile mass reaches tau (the last positive one on rounding)
      int c = cA;
      while (c < last && sCum[c] < tau) ++c;
      const double run = c > cA ? sCum[c - 1] : 0.0;
      const double tau_c = (tau - run) * exp2((double)sTM[t] - (double)sCs[c].x);
      sChunk[i] = c;
      sTl[i] = nextafterf(__double2float_ru(tau_c), -INFINITY);  // P[k] >= tau_c
      sWt[i] = sTW[t];
    }
  }
  __syncthreads();

  gather_chunk_rows<T, D, true>(p, b, h, rank, kvh, bh, Sl, m_lo, seqlen, sChunk, sTl, sRed, sPart, sWt, Mmax);
  return sPart;
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kSampleThreads, 1) flash_gather_kernel(SampleParams p, int CPT, int Mmax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  namespace cg = cooperative_groups;
  const int CS = p.cluster;
  const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int h = blockIdx.x / CS, b = blockIdx.y;
  const size_t bh = (size_t)b * p.H + h;
  float* sPart = flash_item<T, D, G>(p, b, h, rank, CS, CPT, Mmax, smem_raw);
  finish_head<T, D>(p, bh, rank, CS, sPart, 1.0f);  // the merge weights already carry 1 / (Z S_tile)
}

}  // namespace santa
