// step_kernel.cuh -- the whole SANTA decode step in ONE pipelined persistent launch, with no
// gpu-scope fences (the global dependency of sampling, is
// resolved per (b, kv-head) unit instead of per grid).
//
// One CTA per SM (cooperative launch: co-residency is guaranteed, which the polling below relies
// on), three warp roles:
//   * producer (1 warp, one lane): TMA ring as in score_stream_body, but the chunks are
//     INTERLEAVED over the grid -- CTA i takes global chunks w = i, i + grid, i + 2 grid, ...
//     (w = unit * Cmax + c, unit = b * Hkv + kv-head).  Every CTA walks the units in the same
//     order, so unit u is fully scored after ~(u+1)/(B Hkv) of the stream (and the interleaved
//     order streams ~7% faster, tools/microbench_b2b.cu).
//   * NW consumer warps: the score stage of score_stream_body (mma.sync over the swizzled stage,
//     register epilogue), publishing each chunk's results as SELF-VALIDATING words (below).
//   * NSW sampler warps: work items (b, h, split r of CS), unit-major, item t on CTA t % grid.
//     Thresholds (Philox) first; then the group polls its unit's chunk records until every one
//     carries this launch's tag, and runs the combine (fp64 chunk CDF), the inverse CDF and the
//     gather-add.  Unit u's sampling overlaps the streaming of units > u.
//
// Why tagged words instead of counters + fences: publishing through a counter needs a gpu-scope
// release fence after the data stores; with ~200 KB of TMA loads in flight per SM every such
// fence drains them (~1 us each, +4.5 us per step at config 2; tools/microbench_step.cu).  Like
// NCCL's LL protocol, each datum is instead written together with a per-launch tag in ONE
// single-copy-atomic store, and readers poll until the tag matches:
//   * chunk record  [B,H,Cmax] x 16 B: two 64-bit words {m_c | tag32 << 32, l_c | tag32 << 32}
//   * prefix stash  [B,H,Cmax,32] x 8 B: tag16 << 48 | q_{2i+1} << 24 | q_{2i}, q = rn(P_c[k] / l_c *
//     (2^24 - 1)) (the in-chunk prefix as 24-bit fixed point of the chunk's mass, two keys per
//     word: DESIGN.md reading #23)
//   * split partial [B,H,CS,D] x 8 B: {fp32 bits | tag32 << 32}
// tag32 = epoch + 1, tag16 = epoch % 65535 + 1, where epoch is a workspace word read by every CTA at
// start and bumped by the last CTA to exit (an exit ticket; the next launch is stream-ordered
// after it).  CS > 1 splits of a head are summed in fixed split order by the split that draws
// the last ticket (deterministic, no float atomics).  The workspace flag word is written by CTA 0
// at start (SANTA_FLAG_EMPTY_SEQ from seqlens); only the timeout bit is OR-ed in later.
// Polls give up after ~0.5 s and raise SANTA_FLAG_SYNC_TIMEOUT (never a hang).
#pragma once
#include "sample_kernels.cuh"
#include "score_kernels.cuh"

namespace santa {

constexpr int kStepConsumers = 6;   // NW
constexpr int kStepSlots = 2;       // SPW
constexpr int kStepStageKeys = 64;  // keys per TMA stage (= the chunk length L)
constexpr int kStepSamplers = 4;    // NSW (sampler warps per CTA)
constexpr int kStepBarrier = 1;     // named barrier id of the sampler group
constexpr int kStepMaxSplits = 16;  // CS limit (workspace split-partial region)
constexpr uint32_t kQMax = 16777215u;  // 2^24 - 1
constexpr int kStepCPT = 8;         // chunks per sampler thread in the chunk-CDF registers
constexpr int kStepMaxChunks = kStepSamplers * 32 * kStepCPT;  // 1024 chunks = 65,536 tokens

struct StepSync {
  uint32_t* epoch;            // [1]  launch epoch (tags), bumped by the last CTA to exit
  uint32_t* exit_ticket;      // [1]  CTAs done (zero at rest)
  uint32_t* head_ticket;      // [B*H] finished splits of the head (zero at rest)
  ulonglong2* rec;            // [B*H*Cmax] chunk records
  uint32_t* stash;            // [B*H*Cmax*64] tagged fixed-point prefix
  unsigned long long* part;   // [B*H*CS*D] tagged split partials
  unsigned long long* trace;  // NULL in the library; tools/microbench_step.cu timeline (globaltimer ns)
};
// trace layout: per CTA kTraceStride words at trace[blockIdx.x * kTraceStride]: [0] start,
// [1] producer done, [2+j] consumer j last chunk done, [14+j] consumer j first stage landed,
// [24 + 10i + k] sampler item i (< 3): k = 0 wait start, 1 wait done, 2 stats loaded, 3 CDF done,
// 4 chunk search done, 5 gather done, 6 out written, 7 item end, 8 stash validated, 9 indices; [64 + 3j + {0,1,2}] consumer j
// summed ns waiting for stages / in LDS+MMA / in the epilogue, [88 + j] consumer j chunks.
constexpr int kTraceStride = 128;
#define STEP_TRACE(slot) \
  if (sy.trace) sy.trace[(size_t)blockIdx.x * kTraceStride + (slot)] = gtimer()

// Tagged-word WRITES are strong too (.relaxed.gpu): the readers poll with strong loads, and a weak
// store racing with a strong load is a data race under the PTX memory model.  Each word is written
// by one single-copy-atomic store, so a reader sees either the old or the new word, never a mix.
__device__ __forceinline__ void st_v2_u64(void* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_u64(void* p, unsigned long long a) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
// Polling loads must be STRONG (.relaxed.gpu): a weak ld (even .cg) may legally be hoisted out of
// a spin loop by ptxas, since nothing in the loop writes memory (observed: the poll never re-read).
__device__ __forceinline__ ulonglong2 ld_strong_v2_u64(const void* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_strong_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_strong_v4_u32(const void* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ bool rec_valid(const ulonglong2& r, uint32_t tag32) {
  return (uint32_t)(r.x >> 32) == tag32 && (uint32_t)(r.y >> 32) == tag32;
}
__device__ __forceinline__ bool poll_expired(unsigned long long t0) { return gtimer() - t0 > 500000000ull; }

__device__ __forceinline__ void group_bar() { named_bar_sync(kStepBarrier, kStepSamplers * 32); }

// ---------------------------------------------------------------------------------------
// Consumer epilogue for one 64-key chunk, all G heads (lane -> head h = lane / LPH, keys
// [KPL r, KPL r + KPL)), as warp_chunk_epilogue's L = 64 path, but publishing tagged words.
template <int G>
__device__ __forceinline__ void warp_chunk_epilogue_ll(const float* sS, int n_valid, uint32_t* stash_h0,
                                                       ulonglong2* rec_h0, int Cmax, uint32_t tag32, uint32_t tag16) {
  constexpr int LPH = 32 / G;
  constexpr int KPL = 64 / LPH;  // 2, 4, 8, 16 for G = 1, 2, 4, 8
  const int lane = threadIdx.x & 31;
  const int h = lane / LPH, r = lane % LPH;
  const int k0 = r * KPL;
  const float* s = sS + h * 64 + k0;
  float v[KPL];
  if constexpr (KPL >= 4) {
#pragma unroll
    for (int i = 0; i < KPL / 4; ++i) {
      const float4 x = *reinterpret_cast<const float4*>(s + 4 * i);
      v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
    }
  } else {
    const float2 x = *reinterpret_cast<const float2*>(s);
    v[0] = x.x; v[1] = x.y;
  }
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    if (k0 + i >= n_valid) v[i] = -INFINITY;
    m = fmaxf(m, v[i]);
  }
#pragma unroll
  for (int o = LPH / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float ms = (m == -INFINITY) ? 0.f : m;
#pragma unroll
  for (int i = 0; i < KPL; ++i) v[i] = ex2(v[i] - ms);
#pragma unroll
  for (int i = 1; i < KPL; ++i) v[i] += v[i - 1];
  const float tot = v[KPL - 1];
  float incl = tot;
#pragma unroll
  for (int o = 1; o < LPH; o <<= 1) {
    const float t = __shfl_up_sync(0xffffffffu, incl, o);
    if (r >= o) incl += t;
  }
  const float excl = incl - tot;
  const float total = __shfl_sync(0xffffffffu, incl, h * LPH + LPH - 1);
  const float sc = (float)kQMax / total;  // total >= 1 (the max key contributes 2^0)
  const unsigned long long tg = (unsigned long long)tag16 << 48;
  unsigned long long q[KPL / 2];  // two 24-bit keys + the 16-bit tag per word
#pragma unroll
  for (int i = 0; i < KPL / 2; ++i)
    q[i] = tg | ((unsigned long long)min(kQMax, __float2uint_rn((v[2 * i + 1] + excl) * sc)) << 24) |
           (unsigned long long)min(kQMax, __float2uint_rn((v[2 * i] + excl) * sc));
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(stash_h0 + (size_t)h * Cmax * 64 + k0);
  if constexpr (KPL >= 4) {
#pragma unroll
    for (int i = 0; i < KPL / 2; i += 2)  // two independently tagged 64-bit words per 16-B store
      st_v2_u64(dst + i, q[i], q[i + 1]);
  } else {
    st_u64(dst, q[0]);
  }
  if (r == 0) {
    const unsigned long long t = (unsigned long long)tag32 << 32;
    st_v2_u64(rec_h0 + (size_t)h * Cmax, t | __float_as_uint(m), t | __float_as_uint(total));
  }
}

// ---------------------------------------------------------------------------------------
// Sampler-group item: (b, h, split rank of CS), 64-key chunks.  Arithmetic as sample_item
// (readings #1-#5, #21) except the in-chunk search, which runs on the 24-bit fixed-point prefix
// (reading #23).  Returns the partial sum (not yet x 1/S) in sPart[D].
template <typename T, int D, int G, int U = 8>
__device__ float* step_sample_item(const SampleParams& p, const StepSync& sy, int b, int h, int rank, int CS,
                                   unsigned char* smem, int tslot, uint32_t tag32, uint32_t tag16, bool dry) {
  constexpr int NT = kStepSamplers * 32, NW = kStepSamplers, NHW = NT / 16;
  const int tid = threadIdx.x - (blockDim.x - NT);  // 0..NT-1 within the group
  const int lane = tid & 31, wg = tid >> 5;
  const int kvh = h / G;
  const size_t bh = (size_t)b * p.H + h;
  const int S = p.S;
  const int m_lo = (int)((long long)S * rank / CS), m_hi = (int)((long long)S * (rank + 1) / CS);
  const int Sl = m_hi - m_lo;
  const int Slmax = (S + CS - 1) / CS;
  double* sF = reinterpret_cast<double*>(smem);          // [Cmax] chunk CDF
  double* sT = sF + p.Cmax;                              // [Slmax] thresholds
  double* sR = sT + Slmax;                               // [Cmax] W_c (chunk weight, scale 2^-m*)
  int* sChunk = reinterpret_cast<int*>(sR + p.Cmax);     // [Slmax]
  uint32_t* sTq = reinterpret_cast<uint32_t*>(sChunk + Slmax);  // [Slmax] fixed-point threshold
  float* sRed = reinterpret_cast<float*>(sTq + Slmax);   // [NHW][D]
  float* sPart = sRed + NHW * D;                         // [D]
  __shared__ double gred_d[NW];
  __shared__ float gred_f[NW];
  __shared__ int gred_i[NW];
  __shared__ double gZ;

  // ---- a4: thresholds, before waiting (overlaps the score stream) ----
  {
    PhiloxStream ps(p.seed, p.offset, kTagValueSampler, (uint32_t)(p.head_offset + h), (uint32_t)(p.batch_offset + b));
    for (int i = tid; i < Sl; i += NT) sT[i] = sample_threshold(p.mode, m_lo + i, S, ps);
  }
  const int seqlen = __ldg(p.seqlens + b);
  const int nC = seqlen > 0 ? min((seqlen + 63) / 64, p.Cmax) : 0;
  if (tid == 0 && tslot >= 0) STEP_TRACE(tslot + 0);
  if (nC == 0) {  // empty distribution: zero partial (the flag was set at kernel start)
    for (int d = tid; d < D; d += NT) sPart[d] = 0.f;
    if (p.idx_out && !dry)
      for (int i = tid; i < Sl; i += NT) p.idx_out[bh * S + m_lo + i] = -1;
    group_bar();
    return sPart;
  }
  const ulonglong2* rec = sy.rec + bh * p.Cmax;
  // ---- wait: one thread polls the unit's last chunk (it is scored last) with a short back-off, so
  // the ~10^4 waiting sampler threads of a step do not flood L2 while the stream runs ----
  if (tid == 0) {
    const unsigned long long t0 = gtimer();
    while (!rec_valid(ld_strong_v2_u64(rec + nC - 1), tag32)) {
      if (poll_expired(t0)) {
        atomicOr(p.flags, SANTA_FLAG_SYNC_TIMEOUT);
        break;
      }
      __nanosleep(64);
    }
    if (tslot >= 0) STEP_TRACE(tslot + 1);
  }
  group_bar();

  // ---- a3: chunk records -> fp64 chunk CDF (reading #5 clamp), values kept in registers ----
  constexpr int kCPT = kStepCPT;              // chunks per thread (Cmax <= kStepMaxChunks, host-checked)
  const int per = (nC + NT - 1) / NT;         // <= kCPT
  const int c0 = min(tid * per, nC);
  const int nmine = min(per, nC - c0);
  float mreg[kCPT], lreg[kCPT];
  float mloc = -INFINITY;
  {
    ulonglong2 r[kCPT];
#pragma unroll
    for (int i = 0; i < kCPT; ++i)
      if (i < nmine) r[i] = ld_strong_v2_u64(rec + c0 + i);  // one round trip for all of them
    const unsigned long long t0 = gtimer();
#pragma unroll
    for (int i = 0; i < kCPT; ++i) {
      mreg[i] = -INFINITY;
      lreg[i] = 0.f;
      if (i < nmine) {
        while (!rec_valid(r[i], tag32)) {  // rare: a record not yet visible
          if (poll_expired(t0)) {
            atomicOr(p.flags, SANTA_FLAG_SYNC_TIMEOUT);
            break;
          }
          r[i] = ld_strong_v2_u64(rec + c0 + i);
        }
        mreg[i] = __uint_as_float((uint32_t)r[i].x);
        lreg[i] = __uint_as_float((uint32_t)r[i].y);
        mloc = fmaxf(mloc, mreg[i]);
      }
    }
  }
  mloc = warp_max(mloc);
  if (lane == 0) gred_f[wg] = mloc;
  group_bar();
  if (tid == 0 && tslot >= 0) STEP_TRACE(tslot + 2);
  float mstar = gred_f[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) mstar = fmaxf(mstar, gred_f[w]);
  // W_c = 2^(m_c - m*) l_c: the power in fp32 (ex2.approx, 2 ulp) -- the fp32 scores already carry
  // errors of that order -- and everything downstream (products, sums, CDF) in fp64
  // W_c in fp32 (<= 1.5e-7 relative: the ex2 and one rounding), sums and the CDF in fp64
  float wv[kCPT];
  double part = 0.0;
  int lastpos = -1;
#pragma unroll
  for (int i = 0; i < kCPT; ++i) {
    wv[i] = lreg[i] > 0.f ? ex2(mreg[i] - mstar) * lreg[i] : 0.f;
    if (wv[i] > 0.f) lastpos = c0 + i;
  }
#pragma unroll
  for (int i = 0; i < kCPT; ++i) part += (double)wv[i];
  if (sy.trace && tid == 0 && tslot >= 0) sy.trace[(size_t)blockIdx.x * kTraceStride + 120 + (tslot - 24) / 10 * 2] = gtimer();
  {
    const double incl = warp_incl_scan_d(part, lane);
    int lp = lastpos;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lp = max(lp, __shfl_xor_sync(0xffffffffu, lp, o));
    if (lane == 31) gred_d[wg] = incl;
    if (lane == 0) gred_i[wg] = lp;
    group_bar();
    if (sy.trace && tid == 0 && tslot >= 0) sy.trace[(size_t)blockIdx.x * kTraceStride + 121 + (tslot - 24) / 10 * 2] = gtimer();
    double off = 0.0, Z = 0.0;
    int lpos = -1;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const double x = gred_d[w];
      if (w < wg) off += x;
      Z += x;
      lpos = max(lpos, gred_i[w]);
    }
    double run = off + incl - part;
    const double invZ = 1.0 / Z;
#pragma unroll
    for (int i = 0; i < kCPT; ++i) {
      if (i < nmine) {
        run += (double)wv[i];
        sF[c0 + i] = c0 + i >= lpos ? 1.0 : run * invZ;
        sR[c0 + i] = (double)wv[i];
      }
    }
    if (tid == 0) gZ = Z;
  }
  group_bar();
  if (tid == 0 && tslot >= 0) STEP_TRACE(tslot + 3);

  // ---- a5 (part 1): chunk of every sample + its fixed-point in-chunk threshold ----
  for (int m = tid; m < Sl; m += NT) {
    const double Tm = sT[m];
    int lo = 0, hi = nC - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sF[mid] > Tm) hi = mid; else lo = mid + 1;
    }
    const double Fprev = lo ? sF[lo - 1] : 0.0;
    // (T - F_{c-1}) Z / W_c in units of 2^-24 of the chunk's mass (one fp64 division per sample)
    const double tq = (Tm - Fprev) * gZ * (double)kQMax / sR[lo];
    sChunk[m] = lo;
    sTq[m] = tq <= 0.0 ? 0u : (tq >= (double)kQMax ? kQMax : (uint32_t)tq);
  }
  group_bar();
  if (tid == 0 && tslot >= 0) STEP_TRACE(tslot + 4);

  // ---- a5 (part 2) + a6: half-warp per sample: in-chunk count + gather-add ----
  constexpr int EB = (int)sizeof(T);
  constexpr int VCH = D * EB / 16;
  constexpr int NCH = (VCH + 15) / 16;
  constexpr int EPC = 16 / EB;
  // U samples in flight per half-warp (8 half-warps x U strata per round)
  const int hw = tid >> 4, l = tid & 15;
  const unsigned hmask = 0xffffu << (tid & 16);
  float acc[NCH][EPC];
#pragma unroll
  for (int qq = 0; qq < NCH; ++qq)
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[qq][e] = 0.f;
  const T* Vb = reinterpret_cast<const T*>(p.V);
  const uint32_t* Qbase = sy.stash + bh * (size_t)p.Cmax * 64;
  // V row address: contiguous caches hoist the (b, kv-head) base (one multiply-add per row; the
  // generic paged/contiguous KvLayout::row() inlined per sample serialised the loads' issue)
  const T* vbase = p.kv.page_table ? Vb : Vb + ((int64_t)b * p.kv.n_kv_heads + kvh) * p.kv.page_size * D;
  auto vrow = [&](int t) -> const T* {
    return p.kv.page_table ? Vb + p.kv.row(b, kvh, t, D) : vbase + (int64_t)t * D;
  };
  const uint32_t tg16 = tag16;
  const unsigned long long tfull = ((unsigned long long)tag16 << 48) | ((unsigned long long)kQMax << 24) | kQMax;
  for (int mw = 2 * wg; mw < Sl; mw += NHW * U) {
    const int m0 = mw + (hw & 1);
    int jj[U];
    ulonglong2 pv[U];  // lane l: keys 4l, 4l+1 (x) and 4l+2, 4l+3 (y)
    int cc[U], nn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + u * NHW;
      cc[u] = m < Sl ? sChunk[m] : -1;
      nn[u] = cc[u] >= 0 ? min(64, seqlen - cc[u] * 64) : 0;
      pv[u] = make_ulonglong2(tfull, tfull);
      if (cc[u] >= 0) pv[u] = ld_strong_v2_u64(Qbase + (size_t)cc[u] * 64 + 4 * l);  // all 32 words are written
    }
    // validate the tags of every loaded word; re-load the stale ones (warp-uniform loop)
    {
      const unsigned long long t0 = gtimer();
      for (;;) {
        bool bad = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const ulonglong2 v = pv[u];
          if (cc[u] >= 0 && ((uint32_t)(v.x >> 48) != tg16 || (uint32_t)(v.y >> 48) != tg16)) {
            bad = true;
            pv[u] = ld_strong_v2_u64(Qbase + (size_t)cc[u] * 64 + 4 * l);
          }
        }
        if (!__any_sync(0xffffffffu, bad)) break;
        if (poll_expired(t0)) {
          if (l == 0) atomicOr(p.flags, SANTA_FLAG_SYNC_TIMEOUT);
          break;
        }
      }
    }
    if (tid == 0 && tslot >= 0 && mw == 0) STEP_TRACE(tslot + 8);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = m0 + u * NHW;
      const bool on = cc[u] >= 0;
      const uint32_t tq = on ? sTq[m] : 0u;
      const ulonglong2 v = pv[u];
      const int kb = 4 * l, n = nn[u];
      // k1 = #{k < n : q[k] <= tq} = min{k : q[k] > tq}; k2 = #{k < n : q[k] < qmax} = the first key
      // reaching the chunk's full mass (used when rounding puts tq at/after it)
      // q is non-decreasing over the chunk's keys (words of keys >= n hold the full mass kQMax and
      // are masked to it), so k = #{k : q[k] <= tq} is found with ONE ballot over every lane's last
      // word (lane j's 4 keys are 4j..4j+3) plus the crossing lane's own count of its 4 words.
      // With tq >= the full mass (rounding) the count runs to n; then the last positive-mass key,
      // the first key holding the full mass, is taken instead.
      const uint32_t qx = kb < n ? ((uint32_t)v.x & kQMax) : kQMax;
      const uint32_t qy = kb + 1 < n ? ((uint32_t)(v.x >> 24) & kQMax) : kQMax;
      const uint32_t qz = kb + 2 < n ? ((uint32_t)v.y & kQMax) : kQMax;
      const uint32_t qw = kb + 3 < n ? ((uint32_t)(v.y >> 24) & kQMax) : kQMax;
      const uint32_t tqe = tq < kQMax ? tq : kQMax - 1u;  // q <= tqe <=> q <= tq, except at the full mass
      const int full_lanes = __popc(__ballot_sync(0xffffffffu, qw <= tqe) & hmask);  // lanes entirely <= tq
      const int own = (qx <= tqe) + (qy <= tqe) + (qz <= tqe) + (qw <= tqe);
      const int cross = __shfl_sync(0xffffffffu, own, (tid & 16) + min(full_lanes, 15));
      int k = full_lanes < 16 ? 4 * full_lanes + cross : 64;  // first k with q[k] > tqe
      k = min(k, n - 1);
      jj[u] = -1;
      if (on) {
        jj[u] = cc[u] * 64 + min(k, n - 1);
        if (l == 0 && p.idx_out && !dry) p.idx_out[bh * S + m_lo + m] = jj[u];
      }
    }
    if (tid == 0 && tslot >= 0 && mw == 0) STEP_TRACE(tslot + 9);
    uint4 raw[U][NCH];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int qq = 0; qq < NCH; ++qq) {
        const int ch = l + 16 * qq;
        raw[u][qq] = (jj[u] >= 0 && ch < VCH) ? ldg_nc(vrow(jj[u]) + ch * EPC) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int qq = 0; qq < NCH; ++qq) {
        if constexpr (EB == 2) {
          const uint32_t w[4] = {raw[u][qq].x, raw[u][qq].y, raw[u][qq].z, raw[u][qq].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[qq][2 * e] += Elem<T>::lo(w[e]);
            acc[qq][2 * e + 1] += Elem<T>::hi(w[e]);
          }
        } else {
          acc[qq][0] += __uint_as_float(raw[u][qq].x);
          acc[qq][1] += __uint_as_float(raw[u][qq].y);
          acc[qq][2] += __uint_as_float(raw[u][qq].z);
          acc[qq][3] += __uint_as_float(raw[u][qq].w);
        }
      }
  }
#pragma unroll
  for (int qq = 0; qq < NCH; ++qq) {
    const int ch = l + 16 * qq;
    if (ch < VCH)
#pragma unroll
      for (int e = 0; e < EPC; ++e) sRed[hw * D + ch * EPC + e] = acc[qq][e];
  }
  group_bar();
  if (tid == 0 && tslot >= 0) STEP_TRACE(tslot + 5);
  for (int d = tid; d < D; d += NT) {
    float s = 0.f;
    for (int r = 0; r < NHW; ++r) s += sRed[r * D + d];  // fixed order
    sPart[d] = s;
  }
  group_bar();
  return sPart;
}

// The sampler-group work loop (items it = blockIdx.x + k * grid), shared by the step kernels.
// Sampler warps are the LAST NSW warps of the CTA.
template <typename T, int D, int G, int NSW, int U = 8>
__device__ __forceinline__ void step_sampler_loop(const SampleParams& sp, const StepSync& sy, unsigned char* samp_smem,
                                                  uint32_t tag32, uint32_t tag16) {
  const int grid = gridDim.x;
  const int gtid = threadIdx.x - (blockDim.x - NSW * 32);
  __shared__ uint32_t sTicket;
  const int CS = sp.cluster;
  const int items = sp.B * sp.H * CS;
  const float invS = 1.0f / (float)sp.S;
  for (int it = blockIdx.x, ord = 0; it < items;) {
    const int rank = it % CS, bh = it / CS;
    const int b = bh / sp.H, h = bh - b * sp.H;
    const int tslot = (sy.trace && ord < 3) ? 24 + 10 * ord : -1;
    const float* sPart = step_sample_item<T, D, G, U>(sp, sy, b, h, rank, CS, samp_smem, tslot, tag32, tag16, false);
    if (CS == 1) {
      for (int d = gtid; d < D; d += NSW * 32) store_out<T, D>(sp, (size_t)bh, d, sPart[d] * invS);
    } else {
      const unsigned long long t = (unsigned long long)tag32 << 32;
      for (int d = gtid; d < D; d += NSW * 32) st_u64(sy.part + (size_t)it * D + d, t | __float_as_uint(sPart[d]));
      group_bar();
      if (gtid == 0) sTicket = atomicAdd(sy.head_ticket + bh, 1u);
      group_bar();
      if (sTicket == (uint32_t)(CS - 1)) {  // last split of the head: fixed-order sum of all splits
        if (gtid == 0) sy.head_ticket[bh] = 0u;
        const unsigned long long t0 = gtimer();
        for (int d = gtid; d < D; d += NSW * 32) {
          unsigned long long v[kStepMaxSplits];
#pragma unroll
          for (int r = 0; r < kStepMaxSplits; ++r)  // all loads in flight at once
            if (r < CS) v[r] = ld_strong_u64(sy.part + ((size_t)bh * CS + r) * D + d);
          float s = 0.f;
#pragma unroll
          for (int r = 0; r < kStepMaxSplits; ++r) {
            if (r >= CS) break;
            while ((uint32_t)(v[r] >> 32) != tag32) {  // rare: a partial not yet visible
              if (poll_expired(t0)) {
                atomicOr(sp.flags, SANTA_FLAG_SYNC_TIMEOUT);
                break;
              }
              v[r] = ld_strong_u64(sy.part + ((size_t)bh * CS + r) * D + d);
            }
            s += __uint_as_float((uint32_t)v[r]);  // fixed split order
          }
          store_out<T, D>(sp, (size_t)bh, d, s * invS);
        }
      }
    }
    if (gtid == 0 && tslot >= 0) STEP_TRACE(tslot + 6);
    group_bar();  // sPart / sTicket are rewritten by the next item
    if (gtid == 0 && tslot >= 0) STEP_TRACE(tslot + 7);
    it += grid;
    ++ord;
  }
}

// ---------------------------------------------------------------------------------------
// kVar (tools/microbench_step.cu ablations only; 0 in the library): bit 0 = consumers skip the
// MMA and epilogue (wait + release only), bit 1 = sampler warps exit immediately.
template <typename T, int D, int G, int NW, int SPW, int NSW, int kVar = 0>
__global__ void __launch_bounds__(32 * (NW + 1 + NSW), 1)
    santa_step_kernel(const __grid_constant__ CUtensorMap tmK, ScoreParams p, SampleParams sp, StepSync sy) {
  constexpr int SK = kStepStageKeys;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int NSLOT = NW * SPW;
  constexpr int kBoxBytes = SK * 128;
  constexpr int kStageBytes = (D / 64) * kBoxBytes;
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* sSall = reinterpret_cast<float*>(ring + (size_t)NSLOT * kStageBytes);  // [NW][G][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(sSall + (size_t)NW * G * 64);
  uint64_t* empty = full + NSLOT;
  unsigned char* samp_smem = reinterpret_cast<unsigned char*>(empty + NSLOT);
  __shared__ uint32_t sEpoch;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
    sEpoch = __ldcg(sy.epoch);
    STEP_TRACE(0);
    if (blockIdx.x == 0) {  // the launch's flag word ("empty distribution")
      uint32_t f = 0u;
      for (int b = 0; b < p.B; ++b)
        if (__ldg(p.seqlens + b) < 1) f = SANTA_FLAG_EMPTY_SEQ;
      *sp.flags = f;
    }
  }
  __syncthreads();
  const uint32_t epoch = sEpoch;
  const uint32_t tag32 = epoch + 1u, tag16 = epoch % 65535u + 1u;

  const int total = p.B * p.Hkv * p.Cmax;
  const int grid = gridDim.x;
  // warp j's chunk sequence: w = blockIdx.x + (j + NW t) grid, t = 0, 1, ...
  const int wstep = NW * grid;
  const int step_u = wstep / p.Cmax, step_c = wstep - step_u * p.Cmax;

  if (warp == NW) {
    // ---------------- TMA producer (one lane), one cursor per consumer warp ----------------
    if (lane == 0) {
      prefetch_tmap(&tmK);
      const uint64_t pol = l2_policy_evict_first();
      int w[NW], s[NW], nst[NW], k[NW];
      ChunkWalk cw[NW];
      int live;
#pragma unroll
      for (int j = 0; j < NW; ++j) {
        w[j] = blockIdx.x + j * grid;
        cw[j].init(w[j] < total ? w[j] : 0, p.Cmax);
        s[j] = 0;
        nst[j] = -1;
        k[j] = 0;
      }
      do {
        live = 0;
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          while (w[j] < total && nst[j] <= 0) {
            if (nst[j] == 0) {
              w[j] += wstep;
              cw[j].advance(step_c, step_u, p.Cmax);
            }
            if (w[j] >= total) break;
            const int b = cw[j].unit / p.Hkv;
            const int n_valid = min(64, __ldg(p.seqlens + b) - cw[j].c * 64);
            nst[j] = n_valid > 0 ? (n_valid + SK - 1) / SK : 0;
            s[j] = 0;
          }
          if (w[j] >= total) continue;
          ++live;
          const int slot = j * SPW + (k[j] % SPW);
          const uint32_t ph = (uint32_t)(k[j] / SPW) & 1u;
          if (!mbar_test(&empty[slot], ph ^ 1u)) continue;
          const int t = cw[j].c * 64 + s[j] * SK;
          int32_t row;
          if (p.kv.page_table) {
            const int b = cw[j].unit / p.Hkv, kvh = cw[j].unit - b * p.Hkv;
            const int page = t / p.kv.page_size, within = t - page * p.kv.page_size;
            const int64_t phys = (int64_t)__ldg(p.kv.page_table + (int64_t)b * p.kv.max_pages + page);
            row = (int32_t)((phys * p.Hkv + kvh) * p.kv.page_size + within);
          } else {
            row = cw[j].unit * p.kv.page_size + t;
          }
          mbar_arrive_expect_tx(&full[slot], kStageBytes);
#pragma unroll
          for (int hh = 0; hh < D / 64; ++hh)
            tma_load_2d(ring + slot * kStageBytes + hh * kBoxBytes, &tmK, 64 * hh, row, &full[slot], pol);
          ++k[j];
          if (++s[j] == nst[j]) nst[j] = 0;
        }
      } while (live);
      STEP_TRACE(1);
    }
  } else if (warp < NW) {
    // ---------------- consumers ----------------
    float* sS = sSall + (size_t)warp * G * 64;
    int k = 0;
    int cur_unit = -1, seqlen = 0;
    uint32_t ndone = 0;
    unsigned long long t_wait = 0, t_mma = 0, t_epi = 0, tm1 = 0;
    uint4 qf[D / 64][2];
    ChunkWalk cw;
    const int w0 = blockIdx.x + warp * grid;
    cw.init(w0 < total ? w0 : 0, p.Cmax);
    for (int w = w0; w < total; w += wstep) {
      const int c = cw.c, unit = cw.unit;
      cw.advance(step_c, step_u, p.Cmax);
      const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
      const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
      if (unit != cur_unit) {
        load_q_frag<T, D, G>(reinterpret_cast<const T*>(p.q) + bh0 * D, qf);
        seqlen = __ldg(p.seqlens + b);
        cur_unit = unit;
      }
      const int n_valid = min(64, seqlen - c * 64);
      if (n_valid <= 0) continue;  // past the end of the sequence: never read
      const int nst = (n_valid + SK - 1) / SK;
      for (int s = 0; s < nst; ++s, ++k) {
        const int slot = warp * SPW + (k % SPW);
        const unsigned long long tw0 = sy.trace ? gtimer() : 0ull;
        mbar_wait(&full[slot], (uint32_t)(k / SPW) & 1u);
        if (sy.trace) {
          tm1 = gtimer();
          t_wait += tm1 - tw0;
        }
        if (k == 0 && lane == 0) STEP_TRACE(14 + warp);
        if constexpr ((kVar & 1) != 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
          continue;
        }
        const uint32_t sa = smem_u32(ring + slot * kStageBytes);
        const int g = lane >> 2, tig = lane & 3;
#pragma unroll
        for (int half = 0; half < SK / 32; ++half) {
          uint4 a[2][D / 64][2][2];
#pragma unroll
          for (int t2 = 0; t2 < 2; ++t2) {
            const int r0 = 16 * (2 * half + t2) + g, r1 = r0 + 8;
#pragma unroll
            for (int hh = 0; hh < D / 64; ++hh)
#pragma unroll
              for (int jj = 0; jj < 2; ++jj) {
                const int cch = 2 * tig + jj;
                a[t2][hh][jj][0] = lds128(sa + hh * kBoxBytes + r0 * 128 + ((cch ^ (r0 & 7)) << 4));
                a[t2][hh][jj][1] = lds128(sa + hh * kBoxBytes + r1 * 128 + ((cch ^ (r1 & 7)) << 4));
              }
          }
          if (half == SK / 32 - 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
          }
          float acc[2][D / 64][2][4];
#pragma unroll
          for (int t2 = 0; t2 < 2; ++t2)
#pragma unroll
            for (int hh = 0; hh < D / 64; ++hh)
#pragma unroll
              for (int jj = 0; jj < 2; ++jj) {
                float* ac = acc[t2][hh][jj];
                ac[0] = ac[1] = ac[2] = ac[3] = 0.f;
              }
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
            for (int t2 = 0; t2 < 2; ++t2)
#pragma unroll
              for (int hh = 0; hh < D / 64; ++hh)
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                  const uint4& r0 = a[t2][hh][jj][0];
                  const uint4& r1 = a[t2][hh][jj][1];
                  if (s2 == 0)
                    Mma<T>::run(acc[t2][hh][jj], r0.x, r1.x, r0.y, r1.y, qf[hh][jj].x, qf[hh][jj].y);
                  else
                    Mma<T>::run(acc[t2][hh][jj], r0.z, r1.z, r0.w, r1.w, qf[hh][jj].z, qf[hh][jj].w);
                }
#pragma unroll
          for (int t2 = 0; t2 < 2; ++t2) {
            float sum[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float v = 0.f;
#pragma unroll
              for (int hh = 0; hh < D / 64; ++hh) v += acc[t2][hh][0][e] + acc[t2][hh][1][e];
              sum[e] = v;
            }
            store_tile_scores<G>(sS, 64, s * SK + 16 * (2 * half + t2), n_valid, sum, p.scale_log2);
          }
        }
      }
      __syncwarp();
      if (sy.trace) {
        const unsigned long long t = gtimer();
        t_mma += t - tm1;
        tm1 = t;
      }
      if constexpr ((kVar & 1) == 0)
        warp_chunk_epilogue_ll<G>(sS, n_valid, sy.stash + (bh0 * p.Cmax + c) * 64, sy.rec + bh0 * p.Cmax + c,
                                  p.Cmax, tag32, tag16);
      __syncwarp();
      ++ndone;
      if (sy.trace) t_epi += gtimer() - tm1;
    }
    if (lane == 0 && sy.trace) {
      STEP_TRACE(2 + warp);
      unsigned long long* x = sy.trace + (size_t)blockIdx.x * kTraceStride;
      x[64 + 3 * warp] = t_wait;
      x[65 + 3 * warp] = t_mma;
      x[66 + 3 * warp] = t_epi;
      x[88 + warp] = ndone;
    }
  } else if constexpr ((kVar & 2) == 0) {
    // ---------------- sampler group ----------------
    // 4 samples in flight per half-warp (tools/path_sweep.py, batch 32: S = 256 403 -> 395 us,
    // S = 512 435 -> 419 us; the tcgen05 kernel keeps 8: its S = 64 / 512 points got slower)
    step_sampler_loop<T, D, G, NSW, 4>(sp, sy, samp_smem, tag32, tag16);
  }
  // ---------------- exit ticket: the last CTA out advances the epoch ----------------
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(sy.exit_ticket, 1u) == (uint32_t)(grid - 1)) {
      *sy.exit_ticket = 0u;
      *sy.epoch = epoch + 1u;
    }
  }
}

__host__ inline size_t step_score_smem_bytes(int D, int G, int NW, int SPW) {
  return 1024 + (size_t)NW * G * 64 * 4 + (size_t)NW * SPW * ((size_t)(D / 64) * kStepStageKeys * 128 + 16);
}
// sampler smem: sF, sR [Cmax] fp64 + sT [Slmax] fp64 + sChunk, sTq [Slmax] + sRed [NHW][D] + sPart [D]
__host__ inline size_t step_sample_smem_bytes(int Cmax, int Slmax, int D) {
  return (size_t)Cmax * 16 + (size_t)Slmax * 16 + (size_t)(kStepSamplers * 2 + 1) * D * 4 + 64;
}

}  // namespace santa
