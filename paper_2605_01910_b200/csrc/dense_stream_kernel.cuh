// dense_stream_kernel.cuh -- in-repo exact dense decode attention on tensor cores (the reference
// the SANTA latency is reported against).  Flash-decoding: every chunk of Ld keys of a
// (batch, kv-head) yields an unnormalised partial (m_c, l_c, o_c = sum_k 2^(s_k - m_c) V_k); the
// LSE combine (dense_combine_kernel, the merge of Alg. flash-k2 P:1701-1703 with exact weights)
// forms softmax(q K^T scale) V (Eq. 1).
//
// Same persistent structure as the SANTA score pass (score_kernels.cuh): one TMA producer lane,
// NW consumer warps each owning whole chunks with warp-private ring slots; a stage is 64 keys of
// K AND V (2 x 2 boxes of 64 rows x 128 B, 128B swizzle, 32 KiB at d = 128).  Per stage a
// consumer warp:
//   scores   mma.sync m16n8k16: [16 keys x d] . [d x 8 heads]  (K fragments via LDS.128, the
//            permuted-d trick of the score pass)
//   softmax  online per head in registers (running max / sum across the chunk's stages; the
//            score C-fragment and the output C-fragment hold the same two heads per thread)
//   P.V      mma.sync m16n8k16 with M = d (8 tiles), N = heads, K = 16 keys: A = V^T fragments by
//            ldmatrix.x4.trans straight from the swizzled V stage, B = P^T (bf16) through a
//            per-warp padded shared buffer.
#pragma once
#include "common.cuh"
#include "score_kernels.cuh"
#include "tma.cuh"

namespace santa {

constexpr int kDenseChunkStream = 256;  // keys per dense partial
constexpr int kDenseStageKeys = 32;     // keys per stage (K + V = 16 KiB at d = 128)
constexpr int kDenseWarps = 6;
constexpr int kDenseSlots = 2;
constexpr int kPRow = 40;  // padded bf16 row of the per-warp P buffer (conflict-free B-fragment loads)

struct DenseStreamParams {
  const void* q;
  KvLayout kv;
  const int32_t* seqlens;
  int B, H, Hkv;
  float scale_log2;
  float2* cstats;  // [B, H, Cmax] (m_c, l_c)
  float* opart;    // [B, H, Cmax, D]
  int Cmax;        // chunks of kDenseChunkStream keys
  uint32_t* flags;
};

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

template <typename T, int D, int G, int NW, int SPW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    dense_stream_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                        DenseStreamParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int NSLOT = NW * SPW;
  constexpr int SK = kDenseStageKeys, NT = SK / 16;  // keys and 16-key tiles per stage
  constexpr int kBoxBytes = SK * 128;
  constexpr int kHalf = (D / 64) * kBoxBytes;  // K (or V) bytes of one stage
  constexpr int kStageBytes = 2 * kHalf;
  constexpr int L = kDenseChunkStream;
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
    if (blockIdx.x == 0 && p.flags) *p.flags = 0u;
  }
  for (int i = threadIdx.x; i < NW * 8 * kPRow; i += blockDim.x) sPall[i] = 0;  // padded heads stay 0
  __syncthreads();
  pdl_launch_dependents();

  // chunks interleaved over the grid (as the score pass): warp j of CTA i takes
  // w = i + (j + NW t) * grid, t = 0, 1, ...
  const int total = p.B * p.Hkv * p.Cmax;
  const int grid = gridDim.x;
  const int wstep = NW * grid;
  const int step_u = wstep / p.Cmax, step_c = wstep - step_u * p.Cmax;
  if (warp == NW) {
    // ---------------- TMA producer (one lane), one cursor per consumer warp ----------------
    if (lane == 0) {
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmV);
      const uint64_t pol = l2_policy_evict_first();
      int w[NW], s[NW], nst[NW], k[NW];
      ChunkWalk cw[NW];
      int live = 0;
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
            const int n_valid = min(L, __ldg(p.seqlens + b) - cw[j].c * L);
            nst[j] = n_valid > 0 ? (n_valid + SK - 1) / SK : 0;
            s[j] = 0;
          }
          if (w[j] >= total) continue;
          ++live;
          const int slot = j * SPW + (k[j] % SPW);
          const uint32_t ph = (uint32_t)(k[j] / SPW) & 1u;
          if (!mbar_test(&empty[slot], ph ^ 1u)) continue;
          const int t = cw[j].c * L + s[j] * SK;
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
          unsigned char* dst = ring + slot * kStageBytes;
#pragma unroll
          for (int h = 0; h < D / 64; ++h) {
            tma_load_2d(dst + h * kBoxBytes, &tmK, 64 * h, row, &full[slot], pol);
            tma_load_2d(dst + kHalf + h * kBoxBytes, &tmV, 64 * h, row, &full[slot], pol);
          }
          ++k[j];
          if (++s[j] == nst[j]) nst[j] = 0;
        }
      } while (live);
    }
    return;
  }
  // ---------------- consumers ----------------
  const int g = lane >> 2, tig = lane & 3;
  uint16_t* sP = sPall + (size_t)warp * 8 * kPRow;
  const uint32_t sP_addr = smem_u32(sP);
  int kk = 0, cur_unit = -1, seqlen = 0;
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
    const int n_valid = min(L, seqlen - c * L);
    if (n_valid <= 0) {
      if (lane < G) p.cstats[(bh0 + lane) * p.Cmax + c] = make_float2(-INFINITY, 0.f);
      continue;
    }
    const int nst = (n_valid + SK - 1) / SK;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float o[D / 16][4];
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    for (int s = 0; s < nst; ++s, ++kk) {
      const int slot = warp * SPW + (kk % SPW);
      mbar_wait(&full[slot], (uint32_t)(kk / SPW) & 1u);
      const uint32_t sa = smem_u32(ring + slot * kStageBytes);
      const int key0 = s * SK;  // within the chunk
      // ---- scores (4 tiles of 16 keys) ----
      float sc[NT][4];
#pragma unroll
      for (int tile = 0; tile < NT; ++tile) tile_scores_smem<T, D, G, kBoxBytes>(sa, tile, qf, sc[tile]);
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int tile = 0; tile < NT; ++tile)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = key0 + 16 * tile + g + ((e & 2) ? 8 : 0);
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
      // ---- P = 2^(s - m) -> bf16 in the per-warp buffer [head][key] ----
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
      // last stage of a sequence: V rows past the end may hold non-finite garbage -> zero them
      if (key0 + SK > n_valid) {
        for (int r = max(0, n_valid - key0); r < SK; ++r)
          for (int h = 0; h < D / 64; ++h)
            if (lane < 8) *reinterpret_cast<uint4*>(ring + slot * kStageBytes + kHalf + h * kBoxBytes + r * 128 + lane * 16) =
                              make_uint4(0u, 0u, 0u, 0u);
      }
      __syncwarp();
      // ---- O^T[d][head] += V^T[d][key] . P^T[key][head] ----
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
    // ---- chunk partial ----
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) l_run[e] += __shfl_xor_sync(0xffffffffu, l_run[e], off);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int head = 2 * tig + e;
      if (head < G) {
        float* dst = p.opart + ((bh0 + head) * p.Cmax + c) * D;
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) {
          dst[16 * mt + g] = o[mt][e];
          dst[16 * mt + g + 8] = o[mt][e + 2];
        }
        if (g == 0) p.cstats[(bh0 + head) * p.Cmax + c] = make_float2(m_run[e], l_run[e]);
      }
    }
  }
  pdl_launch_dependents();
}

}  // namespace santa
