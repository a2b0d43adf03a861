// prop_kernels.cuh -- S^2ANTA-prop with largest-remainder tile budgets (
// App. M: Alg. prop-budgets P:1597-1613 and Alg. prop-pass2).
//
// Kernel 1 of the paper (tile statistics m_t, l_t and the u-stash) is the score
// pass already in the library: a tile is one L-key chunk (B_tile = L = 64 up to 512k tokens), its
// stats are the chunk's (m_c, l_c) in log2 units and the u-stash is the chunk's inclusive prefix
// P_c[k] = sum_{k' <= k} 2^(s_k' - m_c) (fp32).
//
// The paper's Kernels 2 and 3 are fused into one launch, one (b, h) per CTA (or per thread-block
// cluster, the CS CTAs splitting the S samples): the "global barrier" of P:176 is the kernel
// boundary after the score pass, which this kernel waits on with griddepcontrol (PDL).
//   budgets  m* = max_t m_t, W_t = 2^(m_t - m*) l_t (fp64), Z = sum W_t (fixed-order block scan),
//            q_t = S W_t / Z, S_t = floor(q_t) + one each to the R = S - sum floor(q_t) tiles of
//            largest fractional part, ties to the lower tile index: the R largest keys
//            (frac quantised to 2^-40 | inverted tile index) by an MSB radix select in shared
//            memory, finished by an exact in-warp rank of the <= 32 boundary keys (a bitonic sort
//            measured 45% of the kernel).  Exclusive scan of S_t -> tile offsets.
//   counts   Alg. prop-pass2's c_n = floor(a0 + p + x) - floor(a0 + p), p = invdelta U_{n-1}, is
//            the number of integers j in (a0 + invdelta U_{n-1}, a0 + invdelta U_n]; so the j-th
//            sample of tile t (j = 1..S_t) is row min{n : U_n >= (j - a0_t) l_t / S_t} (reading #25),
//            found by the same half-warp prefix search as the SANTA sampler (thread per sample picks
//            the tile by binary search over the offsets).  a0_t = Philox(seed, offset, tag 4,
//            global head, global batch), draw t.
//   V        O_h = sum of the S gathered rows (c_n-fold repeats included), out = O_h / S.
#pragma once
#include "sample_kernels.cuh"

namespace santa {

__host__ __device__ inline size_t prop_smem_bytes(int Cmax, int S_local, int D, int nthreads) {
  return (size_t)Cmax * 8 + (size_t)Cmax * 8 + (size_t)(Cmax + 1) * 4 + (size_t)S_local * 8 +
         (size_t)(nthreads / 16 + 1) * D * 4 + 64;
}

template <typename T, int D, int G>
__device__ float* prop_item(const SampleParams& p, int b, int h, int rank, int CS, unsigned char* smem_raw) {
  const int NT = blockDim.x, NHW = NT >> 4;
  const int kvh = h / G;
  const int tid = threadIdx.x;
  const size_t bh = (size_t)b * p.H + h;
  const int S = p.S;
  const int m_lo = (int)((long long)S * rank / CS), m_hi = (int)((long long)S * (rank + 1) / CS);
  const int Sl = m_hi - m_lo;
  const int Slmax = (S + CS - 1) / CS;
  unsigned long long* sKey = reinterpret_cast<unsigned long long*>(smem_raw);  // [Cmax] LR keys
  float2* sCs = reinterpret_cast<float2*>(sKey + p.Cmax);                      // [Cmax] tile stats
  int* sOff = reinterpret_cast<int*>(sCs + p.Cmax);                            // [Cmax + 1]
  int* sChunk = sOff + p.Cmax + 1;                                             // [Slmax]
  float* sTl = reinterpret_cast<float*>(sChunk + Slmax);                       // [Slmax]
  float* sRed = sTl + Slmax;                                                   // [NHW][D]
  float* sPart = sRed + NHW * D;                                               // [D]
  __shared__ double sred_d[32];
  __shared__ float sred_f[32];
  __shared__ int sHist[256], sSel[3], sNcand, sFlag[32];
  __shared__ unsigned long long sCand[32];

  pdl_wait_primary();
  pdl_launch_dependents();  // the next step's PDL-launched score pass may set up meanwhile
  const int seqlen = __ldg(p.seqlens + b);
  if (seqlen < 1) {  // empty distribution: zero output, flag, no sampling
    for (int d = tid; d < D; d += NT) sPart[d] = 0.f;
    if (rank == 0 && tid == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    if (p.idx_out)
      for (int i = tid; i < Sl; i += NT) p.idx_out[bh * S + m_lo + i] = -1;
    __syncthreads();
    return sPart;
  }
  const int nC = (seqlen + p.L - 1) / p.L;

  // ---- Kernel 2: m*, W_t, Z -----------------------------------------------------------------
  const float2* cs = p.cstats + bh * p.Cmax;
  float mloc = -INFINITY;
  for (int c = tid; c < nC; c += NT) {
    const float2 v = __ldcg(cs + c);
    sCs[c] = v;
    mloc = fmaxf(mloc, v.x);
  }
  const float mstar = block_max_f(mloc, sred_f);  // (its barrier also publishes sCs)
  const int per = (nC + NT - 1) / NT;
  const int c0 = min(tid * per, nC), c1 = min(c0 + per, nC);
  auto weight = [&](int c) -> double {  // W_t = 2^(m_t - m*) l_t, fp64
    const float2 st = sCs[c];
    return st.y > 0.f ? exp2((double)st.x - (double)mstar) * (double)st.y : 0.0;
  };
  double part = 0.0;
  for (int c = c0; c < c1; ++c) part += weight(c);
  double Z;
  (void)block_excl_scan_d(part, sred_d, &Z);

  // ---- quotas, floors, largest-remainder keys --------------------------------------------------
  double flsum = 0.0;
  for (int c = c0; c < c1; ++c) {
    const double q = (double)S * weight(c) / Z;
    const double fl = floor(q);
    const double frac = q - fl;
    sOff[c] = (int)fl;
    // frac in [0, 1) quantised to 40 bits (differences below 2^-40 count as ties: lower tile wins),
    // tile index inverted in the low 23 bits so that larger keys = earlier tiles
    sKey[c] = ((unsigned long long)(frac * 1099511627776.0) << 23) | (unsigned long long)(0x7FFFFF - c);
    flsum += fl;
  }
  double flt;
  (void)block_excl_scan_d(flsum, sred_d, &flt);  // (barrier: keys and floors visible)
  const int R = min(max(S - (int)flt, 0), nC);

  if (R > 0) {
    // the R largest keys by MSB radix select (8-bit digits, 63-bit keys): each pass histograms the
    // digit of the keys that match the selected prefix so far and fixes the digit at which the
    // running count from the top reaches `need`; as soon as the boundary bin holds <= 32 keys they
    // are ranked exactly inside one warp.  Keys are unique (tile index in the low bits).
    unsigned long long prefix = 0ull, pmask = 0ull;
    int need = R;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += NT) sHist[i] = 0;
      if (tid == 0) sNcand = 0;
      __syncthreads();
      for (int c = c0; c < c1; ++c) {
        const unsigned long long k = sKey[c];
        if ((k & pmask) == prefix) atomicAdd(&sHist[(int)((k >> shift) & 255ull)], 1);
      }
      __syncthreads();
      if (tid < 32) {  // warp 0: digit d with above(d) < need <= above(d) + hist[d], from the top
        int cnt[8], run = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          cnt[e] = sHist[255 - (tid * 8 + e)];  // lane 0 holds the largest digits
          run += cnt[e];
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += v;
        }
        int above = incl - run;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (above < need && need <= above + cnt[e]) {
            sSel[0] = 255 - (tid * 8 + e);
            sSel[1] = above;
            sSel[2] = cnt[e];
          }
          above += cnt[e];
        }
      }
      __syncthreads();
      const int d = sSel[0];
      need -= sSel[1];
      prefix |= (unsigned long long)d << shift;
      pmask |= 255ull << shift;
      if (sSel[2] == need || sSel[2] <= 32 || shift == 0) break;
      __syncthreads();  // sSel / sHist are rewritten by the next pass
    }
    // selected: keys above the prefix; of those equal to it, all (bin exactly filled) or the `need`
    // largest, ranked in one warp
    const bool all_bin = sSel[2] == need;
    if (!all_bin) {
      for (int c = c0; c < c1; ++c)
        if ((sKey[c] & pmask) == prefix) sCand[atomicAdd(&sNcand, 1)] = sKey[c];
      __syncthreads();
      if (tid < 32) {
        const int nc = sNcand;  // <= 32 (or, at shift 0, unique full keys: <= 1)
        const unsigned long long mine = tid < nc ? sCand[tid] : 0ull;
        int rank = 0;
        for (int i = 0; i < nc; ++i) rank += sCand[i] > mine;
        sFlag[tid] = (tid < nc && rank < need) ? 1 : 0;
      }
      __syncthreads();
    }
    for (int c = c0; c < c1; ++c) {
      const unsigned long long k = sKey[c];
      bool sel = (k & pmask) > prefix;
      if ((k & pmask) == prefix) {
        if (all_bin) sel = true;
        else
          for (int i = 0; i < sNcand; ++i)
            if (sCand[i] == k) sel = sFlag[i] != 0;
      }
      if (sel) sOff[c] += 1;
    }
    __syncthreads();
  }

  // ---- exclusive scan of S_t -> tile offsets ---------------------------------------------------
  double cnt = 0.0;
  for (int c = c0; c < c1; ++c) cnt += (double)sOff[c];
  double tot;
  int off = (int)block_excl_scan_d(cnt, sred_d, &tot);
  for (int c = c0; c < c1; ++c) {
    const int v = sOff[c];
    sOff[c] = off;
    off += v;
  }
  if (tid == 0) sOff[nC] = S;
  __syncthreads();

  // ---- Kernel 3: tile and in-tile threshold of every sample (thread per sample) ---------------
  {
    PhiloxStream ps(p.seed, p.offset, kTagPropTileOffset, (uint32_t)(p.head_offset + h),
                    (uint32_t)(p.batch_offset + b));
    for (int i = tid; i < Sl; i += NT) {
      const int m = m_lo + i;
      int lo = 0, hi = nC - 1;  // t = max{t : off_t <= m}
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sOff[mid] <= m) lo = mid; else hi = mid - 1;
      }
      const int t = lo;
      const int St = sOff[t + 1] - sOff[t];
      const int j = m - sOff[t] + 1;
      const double a0 = ps.uniform((uint32_t)t);
      const double tau = ((double)j - a0) * (double)sCs[t].y / (double)St;
      // U_n >= tau  <=>  P[n] > pred(ru(tau)) for fp32 P: the shared search counts P[k] <= tf
      sChunk[i] = t;
      sTl[i] = nextafterf(__double2float_ru(tau), -INFINITY);
    }
  }
  __syncthreads();

  gather_chunk_rows<T, D>(p, b, h, rank, kvh, bh, Sl, m_lo, seqlen, sChunk, sTl, sRed, sPart);
  return sPart;
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kSampleThreads, 1) prop_gather_kernel(SampleParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  namespace cg = cooperative_groups;
  const int CS = p.cluster;
  const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int h = blockIdx.x / CS, b = blockIdx.y;
  const size_t bh = (size_t)b * p.H + h;
  float* sPart = prop_item<T, D, G>(p, b, h, rank, CS, smem_raw);
  finish_head<T, D>(p, bh, rank, CS, sPart);
}

}  // namespace santa
