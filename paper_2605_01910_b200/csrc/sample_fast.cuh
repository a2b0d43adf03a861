// sample_fast.cuh -- the low-latency sampler of the two-kernel path
// for 64-key chunks.  It computes what sample_item() computes (readings #1-#5, #24): the fp64
// chunk CDF of the softmax, the Philox thresholds, J = min{j : F(j) > T} and the mean of the V
// rows -- scheduled for the latency-bound chain that follows the score pass at small batch:
//
//   stats load -> chunk CDF -> chunk search -> prefix-block load -> in-chunk count -> V row load
//   -> reduction -> store
//
//  * ONE block barrier before the search.  Warp w owns a contiguous block of chunks and builds
//    their cumulative weights relative to its own maximum m_w: e_c = 2^(m_c - m_w) (fp32 ex2),
//    w_c = e_c l_c and the in-warp inclusive prefix L_c (fp64).  After the barrier every warp
//    combines the 8 warp summaries (m_w, total_w) in fp64 -- s_w = 2^(m_w - m*) -- into the warp
//    offsets off_w and Z.  The global unnormalised cumulative mass is C_c = off_w + s_w L_c, so
//    F_c > T  <=>  L_c > y, y = (T Z - off_w) / s_w: a sample picks its warp block among 8
//    offsets, then binary-searches that block's L_c.  No normalised CDF is ever stored.
//  * In-chunk decision in exact fp64: with y' = y - L_{c-1} the key is
//    k = min{k : e_c P_c[k] > y'} -- e_c P_c[k] is a product of two fp32 numbers, exact in fp64,
//    so the comparison carries no rounding beyond that of y' (reading #21's "exact" rule, now
//    without the fp32 rounding of the threshold).
//  * Sample i of the CTA's strata belongs to warp i % 8 for its whole life: the warp's lanes draw
//    the thresholds (before griddepcontrol.wait), search (lane per sample) and hand
//    (chunk, y', e_c) to the half-warp that loads the prefix block and the V row -- by shuffles,
//    with no shared-memory sample tables and no barrier between search and gather.
//  * Cluster reduction: ranks 1..CS-1 store their partial into rank 0's shared memory (DSMEM)
//    behind one cluster barrier; rank 0 sums in rank order.
//
// Deterministic: fixed reduction orders (half-warp pair, warps, ranks), no atomics on data.
// Grid (H * CS, B), clusters of CS CTAs per (b, h), 256 threads.

#pragma once
#include <cooperative_groups.h>

#include "sample_kernels.cuh"
#include "tma.cuh"

namespace santa {

#ifndef SANTA_FAST_THREADS
#define SANTA_FAST_THREADS 256
#endif
constexpr int kFastThreads = SANTA_FAST_THREADS;
constexpr int kFastWarps = kFastThreads / 32;
constexpr int kFastCPT = 8;  // chunks per thread held in registers (nC <= 2048); longer: two passes

// shared memory: sLoc [Cmax] fp64 | sE [Cmax] fp32 | sBlk [blocks per CTA][D] | sRecv [super-blocks][D]
__host__ __device__ inline size_t sample_fast_smem_bytes(int Cmax, int D, int CS, int S) {
  const int nsb = (S + 63) / 64;
  const int nbl = 64 * ((nsb + CS - 1) / CS) / 8;
  return (size_t)Cmax * 8 + (size_t)((Cmax + 3) & ~3) * 4 + (size_t)nbl * D * 4 + (size_t)nsb * D * 4 + 64;
}

__device__ __forceinline__ uint32_t cluster_map_u32(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One round of the warp: up to 4 blocks of 8 strata (block vl's strata were searched by lanes
// 8 vl .. 8 vl + 7).  Per block, half-warp hw gathers the strata at positions hw, hw + 2, hw + 4,
// hw + 6 in that order, the two half-warps' sums are added, and lanes 0..15 store the BLOCK SUM to
// sBlk[block] -- a summation tree fixed by the global strata alone (CS-invariant outputs).
template <typename T, int D>
__device__ __forceinline__ void fast_gather_blocks(const SampleParams& p, int b, int kvh, size_t bh, int seqlen,
                                                   int warp, int m_lo, int m_hi, int nbl, int round, int lane_c,
                                                   double lane_y, float lane_e, float* sBlk) {
  constexpr int EB = (int)sizeof(T);
  constexpr int VCH = D * EB / 16;      // 16-B chunks per V row
  constexpr int NCH = (VCH + 15) / 16;  // chunks per lane
  constexpr int EPC = 16 / EB;          // elements per chunk
  constexpr int U = 4;
  const int lane = threadIdx.x & 31, hw = lane >> 4, l = lane & 15;
  const unsigned hmask = 0xffffu << (lane & 16);
  const T* Vb = reinterpret_cast<const T*>(p.V);
  const T* vbase = p.kv.page_table ? Vb : Vb + ((int64_t)b * p.kv.n_kv_heads + kvh) * p.kv.page_size * D;
  const float* Pbase = p.stash + bh * p.stash_stride;
#pragma unroll 1
  for (int vl = 0; vl < 4; ++vl) {
    const int bl = warp + kFastWarps * (4 * round + vl);  // local block
    if (bl >= nbl) break;                                 // (warp-uniform)
    int cc[U], nn[U], jj[U];
    double yy[U];
    float ee[U];
    float4 pv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int pos = hw + 2 * u, jl = 8 * vl + pos;  // the lane that searched this stratum
      const int m = m_lo + 8 * bl + pos;
      const int c = __shfl_sync(0xffffffffu, lane_c, jl);
      yy[u] = __shfl_sync(0xffffffffu, lane_y, jl);
      ee[u] = __shfl_sync(0xffffffffu, lane_e, jl);
      cc[u] = m < m_hi ? c : -1;
      nn[u] = cc[u] >= 0 ? min(64, seqlen - cc[u] * 64) : 0;
      pv[u] = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
      if (cc[u] >= 0 && 4 * l < nn[u]) pv[u] = ldcg_f4(reinterpret_cast<const float4*>(Pbase + (size_t)cc[u] * 64) + l);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // k = #{k : e P[k] <= y'} (P non-decreasing; keys beyond the sequence load +inf): one ballot
      // over every lane's last key + the crossing lane's own count of its 4 keys
      const bool on = cc[u] >= 0;
      const double e = (double)ee[u], y = on ? yy[u] : -INFINITY;
      const float4 v = pv[u];
      const bool bx = e * (double)v.x <= y, by = e * (double)v.y <= y, bz = e * (double)v.z <= y,
                 bw = e * (double)v.w <= y;
      const int full_lanes = __popc(__ballot_sync(0xffffffffu, bw) & hmask);
      const int own = (int)bx + (int)by + (int)bz + (int)bw;
      const int cross = __shfl_sync(0xffffffffu, own, (lane & 16) + min(full_lanes, 15));
      int k = full_lanes < 16 ? 4 * full_lanes + cross : 64;
      // rounding put y' at/after the chunk's total: the first key reaching the total (the last
      // positive-mass key, reading #5)
      if (__any_sync(0xffffffffu, on && k >= nn[u])) {
        const int ln = max(nn[u] - 1, 0);
        const int src = (lane & 16) + (ln >> 2);
        const float tx = __shfl_sync(0xffffffffu, v.x, src), ty = __shfl_sync(0xffffffffu, v.y, src);
        const float tz = __shfl_sync(0xffffffffu, v.z, src), tw = __shfl_sync(0xffffffffu, v.w, src);
        const float tot = (ln & 3) == 0 ? tx : (ln & 3) == 1 ? ty : (ln & 3) == 2 ? tz : tw;
        const int fl2 = __popc(__ballot_sync(0xffffffffu, v.w < tot) & hmask);
        const int own2 = (v.x < tot) + (v.y < tot) + (v.z < tot) + (v.w < tot);
        const int cross2 = __shfl_sync(0xffffffffu, own2, (lane & 16) + min(fl2, 15));
        if (on && k >= nn[u]) k = fl2 < 16 ? 4 * fl2 + cross2 : nn[u] - 1;
      }
      jj[u] = on ? cc[u] * 64 + min(k, nn[u] - 1) : -1;
      if (on && l == 0 && p.idx_out) p.idx_out[bh * p.S + m_lo + 8 * bl + hw + 2 * u] = jj[u];
    }
    uint4 raw[U][NCH];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        const int ch = l + 16 * q;
        const T* row = p.kv.page_table ? Vb + p.kv.row(b, kvh, max(jj[u], 0), D) : vbase + (int64_t)max(jj[u], 0) * D;
        raw[u][q] = (jj[u] >= 0 && ch < VCH) ? ldg_nc(row + ch * EPC) : make_uint4(0u, 0u, 0u, 0u);
      }
    float acc[NCH][EPC];
#pragma unroll
    for (int q = 0; q < NCH; ++q)
#pragma unroll
      for (int e = 0; e < EPC; ++e) acc[q][e] = 0.f;
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
#pragma unroll
    for (int q = 0; q < NCH; ++q)
#pragma unroll
      for (int e = 0; e < EPC; ++e) acc[q][e] += __shfl_xor_sync(0xffffffffu, acc[q][e], 16);
    if (lane < 16) {
#pragma unroll
      for (int q = 0; q < NCH; ++q) {
        const int ch = lane + 16 * q;
        if (ch < VCH)
#pragma unroll
          for (int e = 0; e < EPC; ++e) sBlk[(size_t)bl * D + ch * EPC + e] = acc[q][e];
      }
    }
  }
}

// p.trace (tools/microbench_fast.cu only; NULL in the library): per CTA 16 globaltimer stamps
#define FAST_TRACE(i) \
  if (p.trace && threadIdx.x == 0) p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (i)] = gtimer()

// The strata split of a head over the CS CTAs of its cluster: whole super-blocks of 64 strata
// (8 blocks of 8), rank r owning super-blocks [nsb r / CS, nsb (r + 1) / CS) -- block / super-block
// boundaries are fixed by the global strata, so the summation tree is the same for every CS.
struct FastSplit {
  int m_lo, m_hi, nbl, sb_lo, nsb_local, nsb;
  __device__ __forceinline__ FastSplit(int S, int rank, int CS) {
    nsb = (S + 63) / 64;
    sb_lo = (int)((long long)nsb * rank / CS);
    const int sb_hi = (int)((long long)nsb * (rank + 1) / CS);
    nsb_local = sb_hi - sb_lo;
    m_lo = 64 * sb_lo;
    m_hi = min(S, 64 * sb_hi);
    nbl = (m_hi - m_lo + 7) / 8;
  }
  // this warp's blocks bl = warp + 8 nu; round rho holds nu in [4 rho, 4 rho + 4) (lane = 8 (nu - 4 rho) + pos)
  __device__ __forceinline__ int rounds(int warp) const {
    const int nnu = nbl > warp ? (nbl - warp + kFastWarps - 1) / kFastWarps : 0;
    return (nnu + 3) / 4;
  }
  __device__ __forceinline__ int stratum(int warp, int round, int lane) const {  // -1 if none
    const int bl = warp + kFastWarps * (4 * round + (lane >> 3));
    const int m = m_lo + 8 * bl + (lane & 7);
    return (bl < nbl && m < m_hi) ? m : -1;
  }
};

struct FastSmem {
  double* sLoc;   // [Cmax] in-warp inclusive prefix of w_c
  float* sE;      // [Cmax] e_c = 2^(m_c - m_w)
  float* sBlk;    // [blocks of this CTA][D] block sums
  float* sRecv;   // [super-blocks of the head][D] super-block sums (rank 0)
  float* sWm;     // [NW]
  double* sWt;    // [NW]
  int* sWl;       // [NW]
};

// Chunk weights of one thread's chunks [c0, c1) relative to its warp's maximum, the warp scan and
// the in-warp inclusive prefix L_c (written to sLoc, e_c to sE).  PER > 0: the (<= PER) chunks in
// registers, one round trip; PER = 0: two passes over global memory (long contexts).
template <int PER>
__device__ __forceinline__ void fast_block_chunks(const float2* cs, int c0, int c1, int lane, const FastSmem& sm,
                                                  float& mw, double& part, double& incl, int& lastpos) {
  constexpr int R = PER > 0 ? PER : 1;
  float2 st[R];
  float mloc = -INFINITY;
  if constexpr (PER == 2) {
    if (c0 + 2 <= c1 && (reinterpret_cast<uintptr_t>(cs + c0) & 15u) == 0) {  // 16-B aligned pair
      const float4 v = __ldcg(reinterpret_cast<const float4*>(cs + c0));
      st[0] = make_float2(v.x, v.y);
      st[1] = make_float2(v.z, v.w);
    } else {
      st[0] = c0 < c1 ? __ldcg(cs + c0) : make_float2(-INFINITY, 0.f);
      st[1] = c0 + 1 < c1 ? __ldcg(cs + c0 + 1) : make_float2(-INFINITY, 0.f);
    }
  } else if constexpr (PER > 0) {
#pragma unroll
    for (int i = 0; i < PER; ++i) st[i] = (c0 + i < c1) ? __ldcg(cs + c0 + i) : make_float2(-INFINITY, 0.f);
  }
  if constexpr (PER > 0) {
#pragma unroll
    for (int i = 0; i < PER; ++i) mloc = fmaxf(mloc, st[i].x);
  } else {
    for (int c = c0; c < c1; ++c) mloc = fmaxf(mloc, __ldcg(cs + c).x);
  }
  mw = warp_max(mloc);
  const float mws = mw == -INFINITY ? 0.f : mw;
  part = 0.0;
  lastpos = -1;
  if constexpr (PER > 0) {
    float ev[PER];
    double wv[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      ev[i] = (c0 + i < c1 && st[i].y > 0.f) ? ex2(st[i].x - mws) : 0.f;
      wv[i] = (double)ev[i] * (double)st[i].y;
      part += wv[i];
      if (wv[i] > 0.0) lastpos = c0 + i;
    }
    incl = warp_incl_scan_d(part, lane);
    double run = incl - part;
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (c0 + i < c1) {
        run += wv[i];
        sm.sLoc[c0 + i] = run;
        sm.sE[c0 + i] = ev[i];
      }
  } else {
    for (int c = c0; c < c1; ++c) {
      const float2 v = __ldcg(cs + c);
      const double w = (double)(v.y > 0.f ? ex2(v.x - mws) : 0.f) * (double)v.y;
      part += w;
      if (w > 0.0) lastpos = c;
    }
    incl = warp_incl_scan_d(part, lane);
    double run = incl - part;
    for (int c = c0; c < c1; ++c) {
      const float2 v = __ldcg(cs + c);
      const float e = v.y > 0.f ? ex2(v.x - mws) : 0.f;
      run += (double)e * (double)v.y;
      sm.sLoc[c] = run;
      sm.sE[c] = e;
    }
  }
}

// The post-wait chain of one CTA.
template <typename T, int D, int G>
__device__ __forceinline__ void fast_body(const SampleParams& p, const FastSmem& sm, int CS, int rank, double T0) {
  constexpr int NW = kFastWarps;
  constexpr int EB = (int)sizeof(T);
  constexpr int VCH = D * EB / 16;
  constexpr int NCH = (VCH + 15) / 16;
  constexpr int EPC = 16 / EB;
  const int h = blockIdx.x / CS, b = blockIdx.y;
  const int kvh = h / G;
  const size_t bh = (size_t)b * p.H + h;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = p.S;
  const FastSplit sp(S, rank, CS);
  const int m_lo = sp.m_lo, m_hi = sp.m_hi, Sl = m_hi - m_lo;
  const PhiloxStream ps(p.seed, p.offset, kTagValueSampler, (uint32_t)(p.head_offset + h), (uint32_t)(p.batch_offset + b));
  FAST_TRACE(2);

  const int seqlen = __ldg(p.seqlens + b);
  if (seqlen < 1) {  // empty distribution: zeros, flag, idx -1 (every rank returns here)
    for (int d = tid; d < D; d += kFastThreads)
      if (rank == 0) store_out<T, D>(p, bh, d, 0.f);
    if (rank == 0 && tid == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    if (p.idx_out)
      for (int i = tid; i < Sl; i += kFastThreads) p.idx_out[bh * S + m_lo + i] = -1;
    if (CS > 1) cluster_wait();  // complete the kernel-start arrive (every rank of the cluster is here)
    return;
  }
  const int nC = min((seqlen + 63) / 64, p.Cmax);

  // ---- a3 (part 1): per warp block of chunks, weights relative to the warp maximum ------------
  // W_c relative to the warp: e_c = 2^(m_c - m_w) in fp32 (ex2.approx, reading #24), e_c l_c and
  // every sum in fp64; thread-sequential inclusive sums, then a warp scan of the thread totals
  const float2* cs = p.cstats + bh * p.Cmax;
  const int per = (nC + kFastThreads - 1) / kFastThreads;
  const int c0 = min(tid * per, nC), c1 = min(c0 + per, nC);
  float mw;
  double part, incl;
  int lastpos;
  if (per <= 2)  // config 2: 512 chunks over 256 threads, one 16-B load per thread
    fast_block_chunks<2>(cs, c0, c1, lane, sm, mw, part, incl, lastpos);
  else if (per <= kFastCPT)
    fast_block_chunks<kFastCPT>(cs, c0, c1, lane, sm, mw, part, incl, lastpos);
  else
    fast_block_chunks<0>(cs, c0, c1, lane, sm, mw, part, incl, lastpos);
  int lp = lastpos;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lp = max(lp, __shfl_xor_sync(0xffffffffu, lp, o));
  if (lane == 31) sm.sWt[warp] = incl;
  if (lane == 0) {
    sm.sWm[warp] = mw;
    sm.sWl[warp] = lp;
  }
  __syncthreads();  // the only barrier before the search
  FAST_TRACE(3);

  // ---- a3 (part 2), per warp (redundantly): warp offsets and Z in fp64 ----------------------
  // lane i < NW: summary of warp block i; s_i = 2^(m_i - m*), W_i = s_i total_i
  const float mi = lane < NW ? sm.sWm[lane] : -INFINITY;
  const double ti = lane < NW ? sm.sWt[lane] : 0.0;
  const int li = lane < NW ? sm.sWl[lane] : -1;
  const float mstar = warp_max(mi);
  const bool pos = ti > 0.0;
  // s_i = 2^(m_i - m*) in fp64 (exp2_fast: the block scale multiplies a whole block's weights, so
  // an fp32 power here shifted every later CDF boundary -- 10x more boundary-exempt index
  // mismatches at 512k, tools/diag512.py), its reciprocal rounded in fp64
  const double si = pos ? exp2_fast((double)mi - (double)mstar) : 0.0;
  const double ri = pos ? __drcp_rn(si) : 0.0;
  const double Wi = si * ti;
  double endi = Wi;  // C at the end of block i: inclusive scan over the NW summary lanes
#pragma unroll
  for (int o = 1; o < NW; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, endi, o);
    if (lane >= o) endi += t;
  }
  const double Z = __shfl_sync(0xffffffffu, endi, NW - 1);
  const double offi = endi - Wi;                   // C before block i
  const unsigned posmask = __ballot_sync(0xffffffffu, pos && lane < NW);
  const int lwarp = posmask ? 31 - __clz(posmask) : 0;  // last block with mass
  const int blk = 32 * per;                        // chunks per warp block
  FAST_TRACE(4);

  // ---- a5 + a6: lane-per-stratum search (4 blocks of 8 per round), block-wise gather ----------
  const int rounds = sp.rounds(warp);
  for (int r = 0; r < rounds; ++r) {
    const int mstr = sp.stratum(warp, r, lane);
    const double Tm = (r == 0 || mstr < 0) ? T0 : sample_threshold(p.mode, mstr, S, ps);
    const double X = Tm * Z;
    // block: the first w whose end exceeds X (clamped to the last block with mass)
    int w = 0;
#pragma unroll
    for (int i = 0; i < NW - 1; ++i) w += __shfl_sync(0xffffffffu, endi, i) <= X ? 1 : 0;
    w = min(w, lwarp);
    const double offw = __shfl_sync(0xffffffffu, offi, w);
    const double rw = __shfl_sync(0xffffffffu, ri, w);
    const int lastw = __shfl_sync(0xffffffffu, li, w);
    int lane_c = 0;
    double lane_y = 0.0;
    float lane_e = 0.f;
    if (mstr >= 0) {
      const double y = (X - offw) * rw;
      const int cb = w * blk, ce = min(cb + blk, nC);
      // min{c in [cb, ce) : L_c > y} (ce if none): quaternary steps (3 independent loads each),
      // then binary; the answer stays in [lo, hi]
      int lo = cb, hi = ce;
      while (hi - lo >= 4) {
        const int q = (hi - lo) >> 2, b1 = lo + q, b2 = lo + 2 * q, b3 = lo + 3 * q;
        const bool g1 = sm.sLoc[b1 - 1] <= y, g2 = sm.sLoc[b2 - 1] <= y, g3 = sm.sLoc[b3 - 1] <= y;
        if (g3) lo = b3;
        else if (g2) { lo = b2; hi = b3 - 1; }
        else if (g1) { lo = b1; hi = b2 - 1; }
        else hi = b1 - 1;
      }
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sm.sLoc[mid] > y) hi = mid; else lo = mid + 1;
      }
      const int c = min(lo, lastw);  // none (rounding) or a zero-mass tail: the block's last positive chunk
      lane_c = c;
      lane_y = y - (c > cb ? sm.sLoc[c - 1] : 0.0);
      lane_e = sm.sE[c];
    }
    if (r == 0) FAST_TRACE(5);
    fast_gather_blocks<T, D>(p, b, kvh, bh, seqlen, warp, m_lo, m_hi, sp.nbl, r, lane_c, lane_y, lane_e, sm.sBlk);
  }
  FAST_TRACE(6);
  __syncthreads();
  FAST_TRACE(7);
  // ---- reduction, fixed by the strata: super-block sum = its 8 block sums in order; the head's sum =
  // its super-block sums in order (ranks 1..CS-1 store theirs into rank 0's shared memory behind one
  // cluster barrier; the writers need not outlive it) ----
  const float invS = 1.0f / (float)S;
  if (CS > 1) cluster_wait();  // pairs with the arrive at kernel start: every CTA of the cluster has started
  for (int t = tid; t < sp.nsb_local * D; t += kFastThreads) {
    const int sl = t / D, d = t - sl * D;
    float s = 0.f;
    for (int k = 0; k < 8 && 8 * sl + k < sp.nbl; ++k) s += sm.sBlk[(size_t)(8 * sl + k) * D + d];
    float* dst = sm.sRecv + (size_t)(sp.sb_lo + sl) * D + d;
    if (rank != 0) st_cluster_f32(cluster_map_u32(smem_u32(dst), 0), s);
    else *dst = s;
  }
  if (CS > 1) cluster_barrier();
  else __syncthreads();
  if (rank == 0)
    for (int d = tid; d < D; d += kFastThreads) {
      float s = 0.f;
      for (int k = 0; k < sp.nsb; ++k) s += sm.sRecv[(size_t)k * D + d];
      store_out<T, D>(p, bh, d, s * invS);
    }
  FAST_TRACE(8);
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(kFastThreads, kFastThreads == 128 ? 5 : 1) sample_fast_kernel(SampleParams p) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NW = kFastWarps;
  const int CS = p.cluster;
  const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int h = blockIdx.x / CS, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = p.S;
  const FastSplit sp(S, rank, CS);
  __shared__ float sWm[NW];
  __shared__ double sWt[NW];
  __shared__ int sWl[NW];
  FastSmem sm;
  sm.sLoc = reinterpret_cast<double*>(smem_raw);
  sm.sE = reinterpret_cast<float*>(sm.sLoc + p.Cmax);
  sm.sBlk = sm.sE + ((p.Cmax + 3) & ~3);
  sm.sRecv = sm.sBlk + (size_t)((64 * ((sp.nsb + CS - 1) / CS)) / 8) * D;
  sm.sWm = sWm;
  sm.sWt = sWt;
  sm.sWl = sWl;
  FAST_TRACE(0);
  // DSMEM may target a CTA only once it has started: arrive now, wait before the first remote store
  if (CS > 1) cluster_arrive_relaxed();
  // ---- a4: thresholds of the warp's first 32 samples (lane per sample), before the wait ----
  const PhiloxStream ps(p.seed, p.offset, kTagValueSampler, (uint32_t)(p.head_offset + h), (uint32_t)(p.batch_offset + b));
  double T0 = 0.0;
  {
    const int m0 = sp.stratum(warp, 0, lane);
    if (m0 >= 0) T0 = sample_threshold(p.mode, m0, S, ps);
  }
  FAST_TRACE(1);
  pdl_wait_primary();
  // the next kernel in the stream (the next layer's score pass, itself waiting on this grid) may
  // launch now: its set-up overlaps this chain (all CTAs of this one-wave grid are resident)
  pdl_launch_dependents();
  fast_body<T, D, G>(p, sm, CS, rank, T0);
}

}  // namespace santa
