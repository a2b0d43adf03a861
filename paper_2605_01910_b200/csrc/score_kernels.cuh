// score_kernels.cuh -- split-KV score pass of the SANTA decode hot path (SURVEY sec. 8(a)
// rows a1-a2; PAPER Alg. prop-pass1 P:1577-1595 is the prior art).
//
// For every chunk of L keys (L a multiple of 64, chosen per problem) of every (batch,
// kv-head), for all G query heads of the GQA group, with s in log2 units (scale * log2 e
// folded in):
//   * chunk statistics (m_c = max_k s_k, l_c = sum_k 2^(s_k - m_c))      [B, H, C] float2
//   * the inclusive prefix P_c[k] = sum_{k'<=k} 2^(s_k' - m_c)          [B, H, C*L] fp32 stash
// The stash is the paper's "score stash" ("negligible bandwidth (1/d_k)"); storing the
// PREFIX makes the inverse CDF a plain search.
//
// Score math (bf16/fp16): [16 keys x d] . [d x G heads] is a dense contraction done with
// mma.sync.m16n8k16 (keys = M, heads = N padded to 8, d = K).  The contraction index d may
// be permuted freely as long as A (K rows) and B (q) use the same permutation, so a thread
// reads whole 16-byte chunks of its rows.
//
// Main kernel (score_stream_kernel): persistent, one CTA per SM.  Warp 8 is a TMA producer
// that streams 64-key x 128-B boxes (128B-swizzled) of K into an mbarrier ring; warps 0-7
// are consumers, each owning whole chunks (see below).  With the 128B swizzle, logical
// 16-B chunk c of row r sits at c ^ (r & 7); each thread reads chunks c = 2*tig + jj of its
// two rows (g, g+8), which makes every quarter-warp LDS.128 conflict-free.  Permutation:
//   half h (64 d's), jj, s (k-step):  kc in {2tig, 2tig+1}   <-> d = 64h + 8(2tig+jj) + 4s + (kc&1)
//                                     kc in {2tig+8, 2tig+9} <-> d = 64h + 8(2tig+jj) + 4s + 2 + (kc&1)
// Fallback kernel (score_chunk_kernel): one CTA per chunk, direct 128-bit loads -- used for
// fp32 caches and paged layouts whose page size is not a multiple of 64.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace santa {

constexpr int kStageKeys = 64;        // keys per TMA stage / per fallback step

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
  int L;                    // chunk length (multiple of 64)
  int stash_stride;         // Cmax * L
  uint32_t* tickets;        // [B * Hkv], zeroed here for the sample kernel
  uint32_t* flags;          // zeroed here
};

// fused KV append (santa_decode_attention_append): the new token's rows k_new / v_new [B, Hkv, D]
// are written into K_w / V_w (the caches K / V, writable) at slot seqlens[b] - 1 by the producer lane
// that streams that slot's stage, before its TMA load.  A separate kernel parameter of its own entry
// point (score_stream_append_kernel), so the plain pass keeps its parameter block.
struct AppendParams {
  const void* k_new;
  const void* v_new;
  void* K_w;
  void* V_w;
};

// ---------------------------------------------------------------------------------------
// chunk epilogue: per head max, 2^(s - m), inclusive prefix (stash), (m_c, l_c).
// sS[h * L + k] holds scores for k < n_valid; entries >= n_valid are ignored (masked).
// Warp w (of nwarps) handles heads w, w + nwarps, ...  (used by the fallback kernels)
template <int G>
__device__ __forceinline__ void chunk_epilogue(const float* sS, int L, int n_valid, int warp, int nwarps,
                                               float* stash_h0, int stash_stride, float2* cstats_h0, int Cmax) {
  const int lane = threadIdx.x & 31;
  for (int h = warp; h < G; h += nwarps) {
    const float* s = sS + h * L;
    float m = -INFINITY;
    for (int k = lane; k < n_valid; k += 32) m = fmaxf(m, s[k]);
    m = warp_max(m);
    const float ms = (m == -INFINITY) ? 0.f : m;
    float carry = 0.f;
    float* dst = stash_h0 ? stash_h0 + (size_t)h * stash_stride : nullptr;
    for (int k0 = 0; k0 < L; k0 += 32) {
      const int k = k0 + lane;
      const float u = k < n_valid ? ex2(s[k] - ms) : 0.f;
      const float incl = warp_incl_scan(u, lane) + carry;
      if (dst) dst[k] = incl;
      carry = __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) cstats_h0[(size_t)h * Cmax] = make_float2(m, carry);
  }
}

// Single-warp epilogue for one chunk, all G heads at once: lane -> (head h = lane / LPH,
// keys [KPL * (lane % LPH), +KPL)), LPH = 32 / G lanes per head.  Max and scan need only
// log2(LPH) shuffle steps.  sS is [G][L] (this warp's private buffer).
// Fast path (L == 64, KPL = 2G): scores in registers via 16-B smem loads, every exp2 issued
// independently, prefix sums in registers, 16-B stash stores.
template <int G>
__device__ __forceinline__ void warp_chunk_epilogue(const float* sS, int L, int n_valid, float* stash_h0,
                                                    int stash_stride, float2* cstats_h0, int Cmax) {
  constexpr int LPH = 32 / G;
  const int lane = threadIdx.x & 31;
  const int h = lane / LPH, r = lane % LPH;
  if (L == 64) {
    constexpr int KPL = 64 / LPH;  // 2, 4, 8, 16 for G = 1, 2, 4, 8
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
    for (int i = 0; i < KPL; ++i) v[i] = ex2(v[i] - ms);  // independent MUFU ops; ex2(-inf) = 0
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
    if (stash_h0) {
      float* dst = stash_h0 + (size_t)h * stash_stride + k0;
      if constexpr (KPL >= 4) {
#pragma unroll
        for (int i = 0; i < KPL / 4; ++i)
          *reinterpret_cast<float4*>(dst + 4 * i) =
              make_float4(v[4 * i] + excl, v[4 * i + 1] + excl, v[4 * i + 2] + excl, v[4 * i + 3] + excl);
      } else {
        *reinterpret_cast<float2*>(dst) = make_float2(v[0] + excl, v[1] + excl);
      }
    }
    if (r == 0) cstats_h0[(size_t)h * Cmax] = make_float2(m, total);
    return;
  }
  // generic L (multiple of 64)
  const int kpl = L / LPH;
  const int k0 = r * kpl;
  const float* s = sS + h * L + k0;
  float m = -INFINITY;
  for (int k = 0; k < kpl; ++k)
    if (k0 + k < n_valid) m = fmaxf(m, s[k]);
#pragma unroll
  for (int o = LPH / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float ms = (m == -INFINITY) ? 0.f : m;
  float tot = 0.f;
  for (int k = 0; k < kpl; ++k) tot += (k0 + k < n_valid) ? ex2(s[k] - ms) : 0.f;
  float incl = tot;  // inclusive scan of lane totals within the head's LPH lanes
#pragma unroll
  for (int o = 1; o < LPH; o <<= 1) {
    const float t = __shfl_up_sync(0xffffffffu, incl, o);
    if (r >= o) incl += t;
  }
  const float total = __shfl_sync(0xffffffffu, incl, h * LPH + LPH - 1);
  float run = incl - tot;
  if (stash_h0) {
    float* dst = stash_h0 + (size_t)h * stash_stride + k0;
    for (int k = 0; k < kpl; k += 2) {
      float2 o;
      run += (k0 + k < n_valid) ? ex2(s[k] - ms) : 0.f;
      o.x = run;
      run += (k0 + k + 1 < n_valid) ? ex2(s[k + 1] - ms) : 0.f;
      o.y = run;
      *reinterpret_cast<float2*>(dst + k) = o;
    }
  }
  if (r == 0) cstats_h0[(size_t)h * Cmax] = make_float2(m, total);
}

// ---------------------------------------------------------------------------------------
// 16 keys x G heads from one swizzled smem stage: rows 16*tile + {g, g+8}.
template <typename T, int D, int G, int BOXB = 8192>
__device__ __forceinline__ void tile_scores_smem(uint32_t stage_addr, int tile, const uint4 (&qf)[D / 64][2],
                                                 float (&acc)[4]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int r0 = 16 * tile + g, r1 = r0 + 8;
  uint4 a[D / 64][2][2];
#pragma unroll
  for (int h = 0; h < D / 64; ++h)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const int c = 2 * tig + jj;
      a[h][jj][0] = lds128(stage_addr + h * BOXB + r0 * 128 + ((c ^ (r0 & 7)) << 4));
      a[h][jj][1] = lds128(stage_addr + h * BOXB + r1 * 128 + ((c ^ (r1 & 7)) << 4));
    }
  acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
#pragma unroll
  for (int h = 0; h < D / 64; ++h)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      Mma<T>::run(acc, a[h][jj][0].x, a[h][jj][1].x, a[h][jj][0].y, a[h][jj][1].y, qf[h][jj].x, qf[h][jj].y);
      Mma<T>::run(acc, a[h][jj][0].z, a[h][jj][1].z, a[h][jj][0].w, a[h][jj][1].w, qf[h][jj].z, qf[h][jj].w);
    }
}

template <typename T, int D, int G>
__device__ __forceinline__ void load_q_frag(const T* qg, uint4 (&qf)[D / 64][2]) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int h = 0; h < D / 64; ++h)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
      qf[h][jj] = g < G ? *reinterpret_cast<const uint4*>(qg + g * D + 64 * h + 8 * (2 * tig + jj))
                        : make_uint4(0u, 0u, 0u, 0u);
}

template <int G>
__device__ __forceinline__ void store_tile_scores(float* sS, int L, int key0, int n_valid, const float (&acc)[4],
                                                  float scale_log2) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int k0 = key0 + g, k1 = k0 + 8;
  const int h0 = 2 * tig;
  if (h0 < G) {
    sS[h0 * L + k0] = k0 < n_valid ? acc[0] * scale_log2 : -INFINITY;
    sS[h0 * L + k1] = k1 < n_valid ? acc[2] * scale_log2 : -INFINITY;
  }
  if (h0 + 1 < G) {
    sS[(h0 + 1) * L + k0] = k0 < n_valid ? acc[1] * scale_log2 : -INFINITY;
    sS[(h0 + 1) * L + k1] = k1 < n_valid ? acc[3] * scale_log2 : -INFINITY;
  }
}

// ---------------------------------------------------------------------------------------
// Persistent streaming score kernel (bf16 / fp16, page size % 64 == 0 or contiguous).
// Work: the CTA's chunks w_k = blockIdx.x + k * gridDim.x, taken in groups of NW; consumer
// warp j owns chunk j of every group and processes it alone (MMA + epilogue, no CTA
// barrier).  Ring slots are WARP-PRIVATE: warp j owns slots [j*SPW, (j+1)*SPW) and consumes
// them strictly in order, so an mbarrier is never waited on more than one phase ahead
// (with shared round-robin slots a fast warp could see a stale parity complete).  The
// producer issues a group's stages round-robin over the warps (round s: stage s of chunks
// 0..NW-1), so all warps stream in parallel for any L.
// dynamic smem: [NW*SPW][D/64][64 rows x 128 B] ring (1024-B aligned) | sS[NW][G][L] | barriers
// 5 consumer warps x 2 slots (A/B builds, profiles/r02/v61_score_stream_ab.txt): config 2 pass 14.5-14.6 vs
// 14.8 us for 6 x 2, config 3 (2 GiB) 339-340 vs 349-351 us; 4 x 3 / 3 x 4 16.4 / 16.5 us; two CTAs per SM
// (3 x 2 / 2 x 3 each) 16.4 / 18.5 us at config 2
#ifndef SANTA_STREAM_NW  // (tools: A/B builds override these)
#define SANTA_STREAM_NW 5
#define SANTA_STREAM_SPW 2
#endif
// PDL prologue (profiles/r02/v73_score_prologue_ab.txt): thread 0 executes griddepcontrol.wait after the
// barrier set-up and zeroes the flag word, the CTA barrier holds every other thread until then (the
// wait makes the preceding grids' writes visible to the whole grid).  Config 2 pass 14.6 -> 13.05 us,
// step 22.6 -> 20.7 us; config 3 pass 341 -> 337 us.  Every thread waiting instead (2) cost the
// config-3 pass 10 % (373 us); 0 = the pre-PDL prologue (tools only, launch without PDL).
#ifndef SANTA_SCORE_PROLOGUE
#define SANTA_SCORE_PROLOGUE 1
#endif
#ifndef SANTA_STREAM_CTAS
#define SANTA_STREAM_CTAS 1  // persistent CTAs per SM
#endif
constexpr int kStreamWarps = SANTA_STREAM_NW;   // default consumer warps (tuned with tools/microbench_score.cu)
constexpr int kStreamSlots = SANTA_STREAM_SPW;  // default ring slots per consumer warp

// Incremental walk over a strided chunk sequence (no divisions in the loop):
// w -> (c = w % Cmax, unit = w / Cmax), w += step.
struct ChunkWalk {
  int c, unit;
  __device__ __forceinline__ void init(int w, int Cmax) {
    unit = w / Cmax;
    c = w - unit * Cmax;
  }
  __device__ __forceinline__ void advance(int step_c, int step_u, int Cmax) {
    c += step_c;
    unit += step_u;
    if (c >= Cmax) {
      c -= Cmax;
      ++unit;
    }
  }
};

// Persistent streaming score kernel.  Consumer warp j owns the chunks
// w = blockIdx.x + (j + NW*i) * gridDim.x and the ring slots [j*SPW, (j+1)*SPW).  The producer
// lane keeps one cursor per warp and, polling every warp's next slot with a non-blocking
// mbarrier.test_wait, issues the next stage for whichever warp has a free slot -- no
// head-of-line blocking behind a slow warp.
template <typename T, int D, int G, int NW, int SPW, int kAblate = 0,  // kAblate: tools/microbench_score only
          bool kAppend = false>  // the fused KV append (santa_decode_attention_append) -- its own instantiation:
                                 // a runtime test in the producer loop cost the plain pass 1.6 us (14.8 -> 16.4)
__device__ __forceinline__ void score_stream_body(const CUtensorMap* tmKp, const ScoreParams& p,
                                                  unsigned char* smem_raw, const AppendParams* ap = nullptr) {
  const CUtensorMap& tmK = *tmKp;
  constexpr int NSLOT = NW * SPW;
  constexpr int kBoxBytes = 64 * 128;
  constexpr int kStageBytes = (D / 64) * kBoxBytes;
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* sSall = reinterpret_cast<float*>(ring + (size_t)NSLOT * kStageBytes);  // [NW][G][L]
  uint64_t* full = reinterpret_cast<uint64_t*>(sSall + (size_t)NW * G * p.L);
  uint64_t* empty = full + NSLOT;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
#if SANTA_SCORE_PROLOGUE == 1
    pdl_wait_primary();
#endif
#if SANTA_SCORE_PROLOGUE != 2
    if (blockIdx.x == 0 && p.flags) *p.flags = 0u;
#endif
  }
#if SANTA_SCORE_PROLOGUE == 2
  // launched with programmatic stream serialization: nothing global is read or written before the
  // preceding kernel has completed (it may have produced q, appended K / V, or still read the
  // workspace); the launch itself and the barrier set-up overlap its tail
  pdl_wait_primary();
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.flags) *p.flags = 0u;
#endif
  __syncthreads();
#ifdef SANTA_SCORE_EARLY_TRIGGER
  pdl_launch_dependents();
#endif

  // chunks interleaved over the grid (7 % faster streaming than contiguous CTA ranges,
  // tools/microbench_b2b.cu): warp j of CTA i takes w = i + (j + NW t) * grid, t = 0, 1, ...
  const int total = p.B * p.Hkv * p.Cmax;
  const int grid = gridDim.x;
  const int wstep = NW * grid;
  const int step_u = wstep / p.Cmax, step_c = wstep - step_u * p.Cmax;
  if (warp == NW) {
    // ---------------- TMA producer (one lane), one cursor per consumer warp ----------------
    if (lane == 0) {
      prefetch_tmap(&tmK);
      const uint64_t pol = l2_policy_evict_first();
      int w[NW], s[NW], nst[NW], k[NW];
      ChunkWalk cw[NW];
      int live = 0;
#pragma unroll
      for (int j = 0; j < NW; ++j) {
        w[j] = blockIdx.x + j * grid;
        cw[j].init(w[j] < total ? w[j] : 0, p.Cmax);
        s[j] = 0;
        nst[j] = -1;  // -1: chunk not yet inspected
        k[j] = 0;
      }
      do {
        live = 0;
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          // skip forward over empty chunks (past the end of their sequence)
          while (w[j] < total && nst[j] <= 0) {
            if (nst[j] == 0) {
              w[j] += wstep;
              cw[j].advance(step_c, step_u, p.Cmax);
            }
            if (w[j] >= total) break;
            const int b = cw[j].unit / p.Hkv;
            const int n_valid = min(p.L, __ldg(p.seqlens + b) - cw[j].c * p.L);
            nst[j] = n_valid > 0 ? (n_valid + kStageKeys - 1) / kStageKeys : 0;
            s[j] = 0;
          }
          if (w[j] >= total) continue;
          ++live;
          const int slot = j * SPW + (k[j] % SPW);
          const uint32_t ph = (uint32_t)(k[j] / SPW) & 1u;
          if (!mbar_test(&empty[slot], ph ^ 1u)) continue;
          const int t = cw[j].c * p.L + s[j] * kStageKeys;
          int32_t row;
          if (p.kv.page_table) {
            const int b = cw[j].unit / p.Hkv, kvh = cw[j].unit - b * p.Hkv;
            const int page = t / p.kv.page_size, within = t - page * p.kv.page_size;
            const int64_t phys = (int64_t)__ldg(p.kv.page_table + (int64_t)b * p.kv.max_pages + page);
            row = (int32_t)((phys * p.Hkv + kvh) * p.kv.page_size + within);
          } else {
            row = cw[j].unit * p.kv.page_size + t;  // contiguous [B*Hkv][max_seqlen] rows
          }
          if constexpr (kAppend) {  // fused append: the new token lands in this stage -> write it first
            const int b = cw[j].unit / p.Hkv;
            const int tnew = __ldg(p.seqlens + b) - 1;
            if (tnew >= t && tnew < t + kStageKeys) {
              const int64_t drow = (int64_t)row + (tnew - t);  // cache row of the new token (pages hold
              const int64_t srow = cw[j].unit;                 // whole 64-key stages: same page)
              const uint4* ks = reinterpret_cast<const uint4*>(ap->k_new) + srow * (D * sizeof(T) / 16);
              const uint4* vs = reinterpret_cast<const uint4*>(ap->v_new) + srow * (D * sizeof(T) / 16);
              uint4* kd = reinterpret_cast<uint4*>(ap->K_w) + drow * (D * sizeof(T) / 16);
              uint4* vd = reinterpret_cast<uint4*>(ap->V_w) + drow * (D * sizeof(T) / 16);
#pragma unroll
              for (int i = 0; i < (int)(D * sizeof(T) / 16); ++i) {
                kd[i] = __ldg(ks + i);
                vd[i] = __ldg(vs + i);
              }
              // the generic-proxy stores of the K row must be visible to this thread's TMA (async proxy)
              asm volatile("fence.proxy.async.global;" ::: "memory");
            }
          }
          mbar_arrive_expect_tx(&full[slot], kStageBytes);
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
            tma_load_2d(ring + slot * kStageBytes + h * kBoxBytes, &tmK, 64 * h, row, &full[slot], pol);
          ++k[j];
          if (++s[j] == nst[j]) {  // chunk fully issued: move this warp's cursor on
            nst[j] = 0;
          }
        }
      } while (live);
    }
    pdl_launch_dependents();  // late trigger: dependents launch as the last CTAs drain
    return;
  }
  // ---------------- consumers: warp `warp` owns chunks blockIdx.x + (warp + NW t) * grid ----------------
  float* sS = sSall + (size_t)warp * G * p.L;
  int k = 0;  // this warp's stage counter (slot = warp*SPW + k % SPW)
  int cur_unit = -1, seqlen = 0;
  uint4 qf[D / 64][2];
  ChunkWalk cw;
  const int w0 = blockIdx.x + warp * grid;
  cw.init(w0 < total ? w0 : 0, p.Cmax);
  for (int w = w0; w < total; w += wstep) {
    const int c = cw.c, unit = cw.unit;
    cw.advance(step_c, step_u, p.Cmax);
    const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
    const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
    if (c == 0 && lane == 0 && p.tickets) p.tickets[unit] = 0u;
    if (unit != cur_unit) {  // rare: a warp's chunks span at most a few (b, kv-head) units
      load_q_frag<T, D, G>(reinterpret_cast<const T*>(p.q) + bh0 * D, qf);
      seqlen = __ldg(p.seqlens + b);
      cur_unit = unit;
    }
    const int n_valid = min(p.L, seqlen - c * p.L);
    if (n_valid <= 0) {
      if (lane < G) p.cstats[(bh0 + lane) * p.Cmax + c] = make_float2(-INFINITY, 0.f);
      continue;
    }
    const int nst = (n_valid + kStageKeys - 1) / kStageKeys;
    for (int s = 0; s < nst; ++s, ++k) {
      const int slot = warp * SPW + (k % SPW);
      mbar_wait(&full[slot], (uint32_t)(k / SPW) & 1u);
      const uint32_t sa = smem_u32(ring + slot * kStageBytes);
      // pull the whole stage into registers, then free the slot before any math
      uint4 a[4][D / 64][2][2];
      {
        const int g = lane >> 2, tig = lane & 3;
#pragma unroll
        for (int tile = 0; tile < 4; ++tile) {
          const int r0 = 16 * tile + g, r1 = r0 + 8;
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int cch = 2 * tig + jj;
              a[tile][h][jj][0] = lds128(sa + h * 8192 + r0 * 128 + ((cch ^ (r0 & 7)) << 4));
              a[tile][h][jj][1] = lds128(sa + h * 8192 + r1 * 128 + ((cch ^ (r1 & 7)) << 4));
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (kAblate == 2) {
        if (a[0][0][0][0].x == 0x12345u) sS[lane] = 1.f;
        continue;
      }
      // 4 tiles x (D/64 x 2) independent accumulator chains of length 2 (MMA latency hiding)
      float acc[4][D / 64][2][4];
#pragma unroll
      for (int tile = 0; tile < 4; ++tile)
#pragma unroll
        for (int h = 0; h < D / 64; ++h)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            float* ac = acc[tile][h][jj];
            ac[0] = ac[1] = ac[2] = ac[3] = 0.f;
          }
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int tile = 0; tile < 4; ++tile)
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const uint4& r0 = a[tile][h][jj][0];
              const uint4& r1 = a[tile][h][jj][1];
              if (s2 == 0)
                Mma<T>::run(acc[tile][h][jj], r0.x, r1.x, r0.y, r1.y, qf[h][jj].x, qf[h][jj].y);
              else
                Mma<T>::run(acc[tile][h][jj], r0.z, r1.z, r0.w, r1.w, qf[h][jj].z, qf[h][jj].w);
            }
#pragma unroll
      for (int tile = 0; tile < 4; ++tile) {
        float sum[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = 0.f;
#pragma unroll
          for (int h = 0; h < D / 64; ++h) v += acc[tile][h][0][e] + acc[tile][h][1][e];
          sum[e] = v;
        }
        store_tile_scores<G>(sS, p.L, s * kStageKeys + 16 * tile, n_valid, sum, p.scale_log2);
      }
    }
    __syncwarp();
    if (kAblate >= 1) continue;
    warp_chunk_epilogue<G>(sS, p.L, n_valid, p.stash ? p.stash + bh0 * p.stash_stride + (size_t)c * p.L : nullptr,
                           p.stash_stride, p.cstats + bh0 * p.Cmax + c, p.Cmax);
    __syncwarp();
  }
  pdl_launch_dependents();
}

template <typename T, int D, int G, int NW, int SPW, int kAblate = 0>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    score_stream_kernel(const __grid_constant__ CUtensorMap tmK, ScoreParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  score_stream_body<T, D, G, NW, SPW, kAblate>(&tmK, p, smem_raw);
}

template <typename T, int D, int G, int NW, int SPW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    score_stream_append_kernel(const __grid_constant__ CUtensorMap tmK, ScoreParams p, AppendParams ap) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  score_stream_body<T, D, G, NW, SPW, 0, true>(&tmK, p, smem_raw, &ap);
}

// ---------------------------------------------------------------------------------------
// Fallback: one CTA (4 warps) per chunk, direct loads.  bf16/f16 via mma.sync (same d
// permutation as the v1 kernel: chunk index 4*jj + tig), fp32 via FMA dot products.
template <typename T, int D, int G>
__global__ void __launch_bounds__(128) score_chunk_kernel(ScoreParams p) {
  extern __shared__ __align__(16) float sSdyn[];  // [G][L]
  pdl_launch_dependents();
  const int c = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (c == 0 && threadIdx.x == 0) {
    if (p.tickets) p.tickets[b * p.Hkv + kvh] = 0u;
    if (b == 0 && kvh == 0 && p.flags) *p.flags = 0u;
  }
  const int n_valid = min(p.L, __ldg(p.seqlens + b) - c * p.L);
  const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
  float2* cst = p.cstats + bh0 * p.Cmax + c;
  if (n_valid <= 0) {
    if (threadIdx.x < G) cst[(size_t)threadIdx.x * p.Cmax] = make_float2(-INFINITY, 0.f);
    return;
  }
  const T* qg = reinterpret_cast<const T*>(p.q) + bh0 * D;
  const T* K = reinterpret_cast<const T*>(p.K);
  if constexpr (sizeof(T) == 2) {
    constexpr int NJ = D / 32;
    const int g = lane >> 2, tig = lane & 3;
    uint32_t qf[NJ][4];
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
      uint4 v = g < G ? *reinterpret_cast<const uint4*>(qg + g * D + 8 * (4 * jj + tig)) : make_uint4(0, 0, 0, 0);
      qf[jj][0] = v.x; qf[jj][1] = v.y; qf[jj][2] = v.z; qf[jj][3] = v.w;
    }
    for (int s0 = 0; s0 < n_valid; s0 += kStageKeys) {
      uint4 kr[2][NJ];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int kl = s0 + 16 * warp + g + 8 * r;
        if (kl < n_valid) {
          const T* row = K + p.kv.row(b, kvh, c * p.L + kl, D);
#pragma unroll
          for (int jj = 0; jj < NJ; ++jj) kr[r][jj] = ldg_stream(row + 8 * (4 * jj + tig));
        } else {
#pragma unroll
          for (int jj = 0; jj < NJ; ++jj) kr[r][jj] = make_uint4(0, 0, 0, 0);
        }
      }
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        Mma<T>::run(acc, kr[0][jj].x, kr[1][jj].x, kr[0][jj].y, kr[1][jj].y, qf[jj][0], qf[jj][1]);
        Mma<T>::run(acc, kr[0][jj].z, kr[1][jj].z, kr[0][jj].w, kr[1][jj].w, qf[jj][2], qf[jj][3]);
      }
      store_tile_scores<G>(sSdyn, p.L, s0 + 16 * warp, n_valid, acc, p.scale_log2);
    }
  } else {
    constexpr int LPR = D / 4, RPW = 32 / LPR;
    const int sub = lane / LPR, l = lane % LPR;
    float qv[G][4];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const float4 v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(qg) + gg * D + 4 * l);
      qv[gg][0] = v.x; qv[gg][1] = v.y; qv[gg][2] = v.z; qv[gg][3] = v.w;
    }
    const int nk = (n_valid + 4 * RPW - 1) / (4 * RPW) * (4 * RPW);
    for (int k = warp * RPW + sub; k < nk; k += 4 * RPW) {
      float acc[G];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) acc[gg] = 0.f;
      if (k < n_valid) {
        const float4 v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(K) +
                                                          p.kv.row(b, kvh, c * p.L + k, D) + 4 * l);
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
          acc[gg] = fmaf(qv[gg][0], v.x, fmaf(qv[gg][1], v.y, fmaf(qv[gg][2], v.z, qv[gg][3] * v.w)));
      }
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) acc[gg] += __shfl_xor_sync(0xffffffffu, acc[gg], o);
        if (l == 0 && k < n_valid) sSdyn[gg * p.L + k] = acc[gg] * p.scale_log2;
      }
    }
  }
  __syncthreads();
  chunk_epilogue<G>(sSdyn, p.L, n_valid, warp, 4, p.stash ? p.stash + bh0 * p.stash_stride + (size_t)c * p.L : nullptr,
                    p.stash_stride, cst, p.Cmax);
}

// ---------------------------------------------------------------------------------------
// Fixed 256-key chunk scorer used by the dense reference kernel (4 warps x 64 keys).
constexpr int kDenseChunk = 256;

template <typename T, int D, int G>
__device__ __forceinline__ void score_chunk_mma(const T* __restrict__ qg, const T* __restrict__ K,
                                                const KvLayout& kv, int b, int kvh, int chunk_start, int n_valid,
                                                float scale_log2, float* sS) {
  constexpr int NJ = D / 32;
  constexpr int TPW = kDenseChunk / 16 / 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  uint32_t qf[NJ][4];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    uint4 v = g < G ? *reinterpret_cast<const uint4*>(qg + g * D + 8 * (4 * jj + tig)) : make_uint4(0, 0, 0, 0);
    qf[jj][0] = v.x; qf[jj][1] = v.y; qf[jj][2] = v.z; qf[jj][3] = v.w;
  }
  uint4 kr[TPW][2][NJ];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int kl = 64 * warp + 16 * i + g + 8 * r;
      if (kl < n_valid) {
        const T* row = K + kv.row(b, kvh, chunk_start + kl, D);
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) kr[i][r][jj] = ldg_stream(row + 8 * (4 * jj + tig));
      } else {
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) kr[i][r][jj] = make_uint4(0u, 0u, 0u, 0u);
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
    store_tile_scores<G>(sS, kDenseChunk, 64 * warp + 16 * i, n_valid, acc, scale_log2);
  }
}

template <int D, int G>
__device__ __forceinline__ void score_chunk_simt(const float* __restrict__ qg, const float* __restrict__ K,
                                                 const KvLayout& kv, int b, int kvh, int chunk_start, int n_valid,
                                                 float scale_log2, float* sS) {
  constexpr int LPR = D / 4, RPW = 32 / LPR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, l = lane % LPR;
  float qv[G][4];
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    const float4 v = *reinterpret_cast<const float4*>(qg + gg * D + 4 * l);
    qv[gg][0] = v.x; qv[gg][1] = v.y; qv[gg][2] = v.z; qv[gg][3] = v.w;
  }
  for (int k = warp * RPW + sub; k < kDenseChunk; k += 4 * RPW) {
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
      if (l == 0) sS[gg * kDenseChunk + k] = k < n_valid ? acc[gg] * scale_log2 : -INFINITY;
    }
  }
}

}  // namespace santa
