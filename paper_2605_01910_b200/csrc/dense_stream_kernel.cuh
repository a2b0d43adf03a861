// dense_stream_kernel.cuh -- in-repo exact dense decode attention on tensor cores (the reference
// the SANTA latency is reported against): split-KV flash-decoding -- balanced
// contiguous splits of the 32-key stages of every (batch, kv-head) unit, each yielding an
// unnormalised partial (m, l, o = sum_k 2^(s_k - m) V_k) per unit segment, merged by an LSE
// combine (the merge of Alg. flash-k2 P:1701-1703 with exact weights) into
// softmax(q K^T scale) V (Eq. 1).
//
// Persistent TMA structure as the SANTA score pass (score_kernels.cuh): one producer lane, NW
// consumer warps with warp-private ring slots; a stage is 32 keys of K AND V (2 x 2 boxes,
// 128B swizzle, 16 KiB at d = 128).  Per stage a consumer warp:
//   scores   mma.sync m16n8k16: [16 keys x d] . [d x 8 heads]  (K fragments via LDS.128, the
//            permuted-d trick of the score pass)
//   softmax  online per head in registers (running max / sum across the warp's stages of a unit;
//            the score C-fragment and the output C-fragment hold the same two heads per thread)
//   P.V      mma.sync m16n8k16 with M = d (8 tiles), N = heads, K = 16 keys: A = V^T fragments by
//            ldmatrix.x4.trans straight from the swizzled V stage, B = P^T (bf16) through a
//            per-warp padded shared buffer.
#pragma once
#include "common.cuh"
#include "score_kernels.cuh"
#include "tma.cuh"

namespace santa {

// 32-key stages, 3 consumer warps x 4 ring slots (192 KiB in flight per SM) below ~4 MiB of K+V per SM:
// config 2 28.0 us vs 29.6-29.9 for 6 x 2, 28.2-28.3 for 5 x 2 / 4 x 3 / 64-key 3 x 2, 29.2 for 64-key 6 x 1, 30.4 for 2 x 6 (A/B builds,
// profiles/r02/v54-v56_dense_ab.txt) -- fewer warps: fewer split partials to merge and less ring contention
#ifndef SANTA_DENSE_SK  // (tools: A/B builds override the three)
#define SANTA_DENSE_SK 32
#define SANTA_DENSE_NW 3
#define SANTA_DENSE_SPW 4
#endif
constexpr int kDenseStageKeys = SANTA_DENSE_SK;  // keys per stage (K + V = 16 KiB at d = 128, 32 keys)
constexpr int kDenseWarps = SANTA_DENSE_NW;
constexpr int kDenseSlots = SANTA_DENSE_SPW;
// >= 4 MiB of K+V per SM (config 3, 4 GiB): 5 warps x 2 slots 631-633 us vs 672-674 for 6 x 2, 646-658 for
// 4 x 3, 674-676 for 3 x 4 (profiles/r02/v62_dense_large_ab.txt; cuDNN SDPA 600 us)
#ifndef SANTA_DENSE_NWL  // (tools: A/B builds override both)
#define SANTA_DENSE_NWL 5
#define SANTA_DENSE_SPWL 2
#endif
constexpr int kDenseWarpsLarge = SANTA_DENSE_NWL, kDenseSlotsLarge = SANTA_DENSE_SPWL;  // >= 4 MiB of K+V per SM
constexpr int kDenseWarpsMax = kDenseWarps > kDenseWarpsLarge ? kDenseWarps : kDenseWarpsLarge;
constexpr int kPRow = kDenseStageKeys + 8;  // padded bf16 row of the per-warp P buffer (conflict-free B loads)

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

template <typename T>
__device__ __forceinline__ uint16_t to_bits16(float x);
template <>
__device__ __forceinline__ uint16_t to_bits16<__nv_bfloat16>(float x) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}
template <>
__device__ __forceinline__ uint16_t to_bits16<__half>(float x) {
  return __half_as_ushort(__float2half_rn(x));
}

// ---------------------------------------------------------------------------------------
// dense_split_kernel: the same per-stage math with BALANCED work.  dense_stream_kernel hands each
// warp whole 256-key chunks interleaved over the grid: at config 2 (1024 chunks, 888 warps) 136
// warps got two chunks and 752 one, so the pass ran at ~58 % of its balanced rate (30.4 us under
// ncu; cuDNN's SDPA 25.9 us).  Here the flattened sequence of 32-key stages of all (b, kv-head)
// units is cut into grid contiguous CTA ranges of equal length (+-1 stage), and a CTA's stages go
// round-robin to its NW consumer warps.  Each warp keeps one online-softmax partial per unit
// segment of its CTA's range and writes it to slot (cta + unit) * NW + warp (disjoint over units:
// the CTAs covering unit u+1 start where those of unit u end); warps with no stage in a segment
// write an empty partial.  dense_split_combine merges, per (b, h), the slots of the CTAs covering
// its unit (exact LSE weights, fixed order).
constexpr int kDenseSplitMaxCtas = 160;

struct DenseSplitParams {
  const void* q;
  KvLayout kv;
  const int32_t* seqlens;
  int B, H, Hkv;
  float scale_log2;
  float* part_o;    // [slots][G][D]
  float2* part_ml;  // [slots][G] (m, l) in log2 units / unnormalised sum
  void* out;        // [B, H, D]
  uint32_t* flags;
};

__device__ __forceinline__ int dense_stages(int seqlen) { return seqlen > 0 ? (seqlen + kDenseStageKeys - 1) / kDenseStageKeys : 0; }

// total stages and, for stage index s, its unit / stage-in-unit: units ordered (b, kv-head)
struct StageWalk {
  int unit, si, left;  // current unit, stage within it, stages left in it
  const int32_t* seqlens;
  int Hkv, nunits;
  __device__ __forceinline__ void init(const int32_t* sl, int B, int hkv, int s) {
    seqlens = sl;
    Hkv = hkv;
    nunits = B * hkv;
    unit = 0;
    int b = 0;
    for (; b < B; ++b) {
      const int n = dense_stages(__ldg(sl + b));
      if (s < n * hkv) break;
      s -= n * hkv;
    }
    if (b >= B) {
      unit = B * hkv;
      si = 0;
      left = 0;
      return;
    }
    const int n = dense_stages(__ldg(sl + b));
    unit = b * hkv + s / n;
    si = s % n;
    left = n - si;
  }
  __device__ __forceinline__ void next() {  // advance one stage (skipping empty units)
    ++si;
    if (--left > 0) return;
    do {
      ++unit;
      si = 0;
      left = unit < nunits ? dense_stages(__ldg(seqlens + unit / Hkv)) : 1;
    } while (left == 0);
  }
};

template <typename T, int D, int G, int NW, int SPW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    dense_split_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       DenseSplitParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int NSLOT = NW * SPW;
  constexpr int SK = kDenseStageKeys, NT = SK / 16;
  constexpr int kBoxBytes = SK * 128;
  constexpr int kHalf = (D / 64) * kBoxBytes;
  constexpr int kStageBytes = 2 * kHalf;
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint16_t* sPall = reinterpret_cast<uint16_t*>(ring + (size_t)NSLOT * kStageBytes);  // [NW][8][kPRow]
  uint64_t* full = reinterpret_cast<uint64_t*>(sPall + (size_t)NW * 8 * kPRow);
  uint64_t* empty = full + NSLOT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
    pdl_wait_primary();  // PDL launch: global memory only after the preceding kernel completed (thread 0
    if (blockIdx.x == 0 && p.flags) *p.flags = 0u;  // waits, the barrier holds the rest: see score_kernels.cuh)
  }
  for (int i = threadIdx.x; i < NW * 8 * kPRow; i += blockDim.x) sPall[i] = 0;
  __syncthreads();
  pdl_launch_dependents();
  // this CTA's contiguous stage range
  int Stot = 0;
  for (int b = 0; b < p.B; ++b) Stot += dense_stages(__ldg(p.seqlens + b)) * p.Hkv;
  const int s_begin = (int)((long long)Stot * blockIdx.x / gridDim.x);
  const int s_end = (int)((long long)Stot * (blockIdx.x + 1) / gridDim.x);
  const int nunits = p.B * p.Hkv;
  if (warp == NW) {
    // ---------------- TMA producer: stage s -> warp (s - s_begin) % NW, in order ----------------
    if (lane == 0 && s_begin < s_end) {
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmV);
      const uint64_t pol = l2_policy_evict_first();
      StageWalk sw;
      sw.init(p.seqlens, p.B, p.Hkv, s_begin);
      int k[NW];
#pragma unroll
      for (int j = 0; j < NW; ++j) k[j] = 0;
      int j = 0;
      for (int s = s_begin; s < s_end; ++s) {
        const int slot = j * SPW + (k[j] % SPW);
        mbar_wait(&empty[slot], ((uint32_t)(k[j] / SPW) & 1u) ^ 1u);
        const int t = sw.si * SK;
        const int b = sw.unit / p.Hkv, kvh = sw.unit - b * p.Hkv;
        int32_t row;
        if (p.kv.page_table) {
          const int page = t / p.kv.page_size, within = t - page * p.kv.page_size;
          const int64_t phys = (int64_t)__ldg(p.kv.page_table + (int64_t)b * p.kv.max_pages + page);
          row = (int32_t)((phys * p.Hkv + kvh) * p.kv.page_size + within);
        } else {
          row = sw.unit * p.kv.page_size + t;
        }
        mbar_arrive_expect_tx(&full[slot], kStageBytes);
        unsigned char* dst = ring + slot * kStageBytes;
#pragma unroll
        for (int h = 0; h < D / 64; ++h) {
          tma_load_2d(dst + h * kBoxBytes, &tmK, 64 * h, row, &full[slot], pol);
          tma_load_2d(dst + kHalf + h * kBoxBytes, &tmV, 64 * h, row, &full[slot], pol);
        }
        ++k[j];
        j = j + 1 == NW ? 0 : j + 1;
        sw.next();
      }
    }
    return;
  }
  // ---------------- consumers: stages s_begin + warp + NW t ----------------
  const int g = lane >> 2, tig = lane & 3;
  uint16_t* sP = sPall + (size_t)warp * 8 * kPRow;
  if (s_begin >= s_end) return;
  StageWalk sw;
  sw.init(p.seqlens, p.B, p.Hkv, s_begin);
  const int u_first = sw.unit;
  int u_last;
  {
    StageWalk se;
    se.init(p.seqlens, p.B, p.Hkv, s_end - 1);
    u_last = se.unit;
  }
  // advance to this warp's first stage
  for (int i = 0; i < warp && s_begin + i < s_end; ++i) sw.next();
  auto write_slot = [&](int u, const float (&o)[D / 16][4], const float (&m_run)[2], const float (&l_run)[2],
                        bool live) {
    const size_t slot = ((size_t)blockIdx.x + u) * NW + warp;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int head = 2 * tig + e;
      if (head < G) {
        float* dst = p.part_o + (slot * G + head) * D;
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) {
          dst[16 * mt + g] = live ? o[mt][e] : 0.f;
          dst[16 * mt + g + 8] = live ? o[mt][e + 2] : 0.f;
        }
        if (g == 0) p.part_ml[slot * G + head] = live ? make_float2(m_run[e], l_run[e]) : make_float2(-INFINITY, 0.f);
      }
    }
  };
  int kk = 0;
  int u_next = u_first;  // next unit whose slot this warp still has to write
  int cur_unit = -1, seqlen = 0;
  uint4 qf[D / 64][2];
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  float o[D / 16][4];
#pragma unroll
  for (int mt = 0; mt < D / 16; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
  for (int s = s_begin + warp; s < s_end; s += NW) {
    const int unit = sw.unit, si = sw.si;
    for (int i = 0; i < NW; ++i) sw.next();  // this warp's next stage
    if (unit != cur_unit) {
      if (cur_unit >= 0) {  // flush the previous unit's partial
        l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 4);
        l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 8);
        l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 16);
        l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], 4);
        l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], 8);
        l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], 16);
        write_slot(cur_unit, o, m_run, l_run, true);
      }
      for (; u_next < unit; ++u_next) write_slot(u_next, o, m_run, l_run, false);  // no stage of mine there
      u_next = unit + 1;
      m_run[0] = m_run[1] = -INFINITY;
      l_run[0] = l_run[1] = 0.f;
#pragma unroll
      for (int mt = 0; mt < D / 16; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
      const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
      load_q_frag<T, D, G>(reinterpret_cast<const T*>(p.q) + ((size_t)b * p.H + (size_t)kvh * G) * D, qf);
      seqlen = __ldg(p.seqlens + b);
      cur_unit = unit;
    }
    const int slot = warp * SPW + (kk % SPW);
    mbar_wait(&full[slot], (uint32_t)(kk / SPW) & 1u);
    ++kk;
    const uint32_t sa = smem_u32(ring + slot * kStageBytes);
    const int key0 = si * SK;
    const int n_valid = seqlen - key0;  // keys of this stage: min(SK, n_valid)
    float sc[NT][4];
#pragma unroll
    for (int tile = 0; tile < NT; ++tile) tile_scores_smem<T, D, G, kBoxBytes>(sa, tile, qf, sc[tile]);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int tile = 0; tile < NT; ++tile)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = 16 * tile + g + ((e & 2) ? 8 : 0);
        float v = sc[tile][e] * p.scale_log2;
        if (key >= n_valid) v = -INFINITY;
        sc[tile][e] = v;
        mx[e & 1] = fmaxf(mx[e & 1], v);
      }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], off));
    }
    float corr[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float mn = fmaxf(m_run[e], mx[e]);
      corr[e] = (m_run[e] == -INFINITY) ? 0.f : ex2(m_run[e] - mn);
      m_run[e] = mn;
      l_run[e] *= corr[e];
    }
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt) {
      o[mt][0] *= corr[0];
      o[mt][2] *= corr[0];
      o[mt][1] *= corr[1];
      o[mt][3] *= corr[1];
    }
    __syncwarp();
#pragma unroll
    for (int tile = 0; tile < NT; ++tile)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int head = 2 * tig + (e & 1);
        const int keyl = 16 * tile + g + ((e & 2) ? 8 : 0);
        const float ms = m_run[e & 1] == -INFINITY ? 0.f : m_run[e & 1];
        const float pv = ex2(sc[tile][e] - ms);
        l_run[e & 1] += pv;
        if (head < G) sP[head * kPRow + keyl] = to_bits16<T>(pv);
      }
    if (n_valid < SK) {  // the sequence's last stage: V rows past the end may be non-finite garbage
      for (int r = max(0, n_valid); r < SK; ++r)
        for (int h = 0; h < D / 64; ++h)
          if (lane < 8)
            *reinterpret_cast<uint4*>(ring + slot * kStageBytes + kHalf + h * kBoxBytes + r * 128 + lane * 16) =
                make_uint4(0u, 0u, 0u, 0u);
    }
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < NT; ++ks) {
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(sP + g * kPRow + 16 * ks + 2 * tig);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(sP + g * kPRow + 16 * ks + 2 * tig + 8);
      const int krow = 16 * ks + ((lane >> 4) & 1) * 8 + (lane & 7);
#pragma unroll
      for (int mt = 0; mt < D / 16; ++mt) {
        const int d = 16 * mt + ((lane >> 3) & 1) * 8;
        const int box = d >> 6, ch = (d & 63) >> 3;
        const uint32_t addr = sa + kHalf + box * kBoxBytes + krow * 128 + ((ch ^ (krow & 7)) << 4);
        uint32_t a0, a1, a2, a3;
        ldsm_x4_trans(addr, a0, a1, a2, a3);
        Mma<T>::run(o[mt], a0, a1, a2, a3, b0, b1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (cur_unit >= 0) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) l_run[e] += __shfl_xor_sync(0xffffffffu, l_run[e], off);
    }
    write_slot(cur_unit, o, m_run, l_run, true);
  }
  for (; u_next <= u_last && u_next < nunits; ++u_next) write_slot(u_next, o, m_run, l_run, false);
}

// first / last CTA of the contiguous split whose range holds stage s (range c = [Stot c / grid,
// Stot (c + 1) / grid))
__device__ __forceinline__ int dense_cta_of_stage(int s, int Stot, int grid) {
  int c = (int)((long long)s * grid / Stot);
  while (c > 0 && (int)((long long)Stot * c / grid) > s) --c;
  while (c + 1 < grid && (int)((long long)Stot * (c + 1) / grid) <= s) ++c;
  return c;
}

// LSE merge of the split partials of one (b, h) in ONE pass over the slots: CTA (h, d-slice)
// of 512 threads = kDQ output coordinates x 16 parts; thread (d, part) runs an online merge over
// its ~nslot/16 slots (all their loads in flight at once: one L2 round trip at config 2's ~114
// slots per head), then the 16 parts are merged in fixed order.  (Round 2: 4 parts per coordinate
// needed two dependent batches of 16 loads; a max pass + weight pass + value pass cost three round
// trips -- 9.4 us under ncu for 120 slots per head.)
// NPART = 512 / D (one CTA per head) when a head has few slots (config 3: ~1-2 CTAs per unit), else 16.
constexpr int kDenseCombineThreads = 512;
template <typename T, int D, int G, int NW, int NPART>
__global__ void __launch_bounds__(kDenseCombineThreads) dense_split_combine(DenseSplitParams p, int grid) {
  constexpr int NTH = kDenseCombineThreads;
  constexpr int kDQ = NTH / NPART;  // output coordinates per CTA
  static_assert(kDQ <= D && D % kDQ == 0, "combine slice");
  __shared__ float sM[NTH], sNum[NTH], sDen[NTH];
  pdl_wait_primary();
  pdl_launch_dependents();  // the next kernel (waiting on this grid itself) may set up meanwhile
  constexpr int NSL = D / kDQ;
  const int h = blockIdx.x / NSL, dsl = blockIdx.x - h * NSL, b = blockIdx.y, tid = threadIdx.x;
  const int kvh = h / G, gh = h - kvh * G;
  const int u = b * p.Hkv + kvh;
  T* out = reinterpret_cast<T*>(p.out) + ((size_t)b * p.H + h) * D + dsl * kDQ;
  const int seqlen = __ldg(p.seqlens + b);
  if (seqlen < 1) {
    for (int d = tid; d < kDQ; d += NTH) out[d] = Elem<T>::from_f(0.f);
    if (tid == 0 && dsl == 0) atomicOr(p.flags, SANTA_FLAG_EMPTY_SEQ);
    return;
  }
  int Stot = 0, Pu = 0;
  for (int bb = 0; bb < p.B; ++bb) {
    const int n = dense_stages(__ldg(p.seqlens + bb));
    if (bb < b) Pu += n * p.Hkv;
    Stot += n * p.Hkv;
  }
  const int nu = dense_stages(seqlen);
  Pu += kvh * nu;
  const int c0 = dense_cta_of_stage(Pu, Stot, grid), c1 = dense_cta_of_stage(Pu + nu - 1, Stot, grid);
  const int nslot = (c1 - c0 + 1) * NW;
  const size_t slot0 = ((size_t)c0 + u) * NW;
  const int dl = tid % kDQ, part = tid / kDQ, d = dsl * kDQ + dl;
  float m = -INFINITY, num = 0.f, den = 0.f;
  constexpr int U = 8;
  for (int i0 = part; i0 < nslot; i0 += NPART * U) {
    float2 ml[U];
    float v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int i = i0 + q * NPART;
      ml[q] = i < nslot ? __ldcg(&p.part_ml[(slot0 + i) * G + gh]) : make_float2(-INFINITY, 0.f);
      v[q] = i < nslot ? __ldcg(p.part_o + ((slot0 + i) * G + gh) * D + d) : 0.f;
    }
    float mb = m;
#pragma unroll
    for (int q = 0; q < U; ++q) mb = fmaxf(mb, ml[q].y > 0.f ? ml[q].x : -INFINITY);
    if (mb > -INFINITY) {
      const float r = m > -INFINITY ? ex2(m - mb) : 0.f;
      num *= r;
      den *= r;
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const float w = ml[q].y > 0.f ? ex2(ml[q].x - mb) : 0.f;
        num = fmaf(w, v[q], num);
        den = fmaf(w, ml[q].y, den);
      }
      m = mb;
    }
  }
  sM[tid] = m;
  sNum[tid] = num;
  sDen[tid] = den;
  __syncthreads();
  if (tid < kDQ) {
    float ms = -INFINITY;
    for (int q = 0; q < NPART; ++q) ms = fmaxf(ms, sM[q * kDQ + tid]);
    float sn = 0.f, sd = 0.f;
    for (int q = 0; q < NPART; ++q) {
      const float mq = sM[q * kDQ + tid];
      const float r = mq > -INFINITY ? ex2(mq - ms) : 0.f;
      sn = fmaf(r, sNum[q * kDQ + tid], sn);
      sd = fmaf(r, sDen[q * kDQ + tid], sd);
    }
    out[tid] = Elem<T>::from_f(sn / sd);
  }
}

}  // namespace santa
