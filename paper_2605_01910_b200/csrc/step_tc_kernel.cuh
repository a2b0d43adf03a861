// step_tc_kernel.cuh -- the single-launch step kernel with the score stage on the 5th-generation
// tensor cores (tcgen05 + TMEM).  Same algorithm, interleaved tile order, tagged-word
// publication and sampler as santa_step_kernel (step_kernel.cuh); only the score stage differs.
//
// Score stage: per 128-key tile of one (b, kv-head) unit,
//   S[128 keys x 16] = K_tile[128 x d] . Q^T[d x 16]   (q of the G heads, rows G..15 zero)
// is ONE dense contraction: M = 128 keys, N = 16 (G <= 8 heads padded), K = d, bf16/fp16 inputs,
// fp32 accumulation in TMEM.  Operands come straight from the TMA-landed shared-memory stage
// (K-major, 128B swizzle, the same boxes the mma.sync consumers read): the A descriptor points at
// the K tile, the B descriptor at the stage's q rows (TMA-loaded with the tile).  d/16 MMAs per
// tile are issued by ONE thread; tcgen05.commit arrives on the stage's "empty" barrier (the TMA
// producer may refill it) and on the accumulator's "full" barrier.  Warp roles:
//   warps 0-7   two epilogue groups (EG) of 4 warps: tiles alternate between the EGs; each warp
//               reads its TMEM lane quadrant (32 keys x G heads, tcgen05.ld.32x32b), releases the
//               accumulator, writes scaled scores to shared memory; two warps then run the
//               64-key chunk epilogue (max, exp2, prefix, tagged publication) for the tile's 2 chunks
//   warp 8      TMA producer (one lane): K tile (4 boxes of 64 rows x 128 B) + q rows per stage
//   warp 9      MMA issuer (one lane) and TMEM allocator (the warp); warps 10-11 idle
//   warps 12-15 the sampler group (step_sampler_loop)
// Registers are rebalanced per warpgroup with setmaxnreg (512 threads x 128 at launch): the
// producer/MMA warpgroup drops to 56, the epilogue groups to 112, the sampler group grows to 200
// (at 128 it spilled and needed 4-sample rounds; config 3, S = 512 was sampler-bound).
// TMEM: 4 accumulator buffers x 16 columns (64 columns allocated).  Paged caches need pages of a
// multiple of 128 tokens (a tile never straddles pages).
#pragma once
#include <type_traits>

#include "step_kernel.cuh"

namespace santa {

constexpr int kTcTileKeys = 128;  // MMA M (keys per tile = 2 chunks)
constexpr int kTcN = 16;          // MMA N (heads padded)
constexpr int kTcStages = 5;      // smem ring stages (one tile each)
constexpr int kTcBufs = 4;        // TMEM accumulator buffers
constexpr int kTcCols = 64;       // TMEM columns allocated (kTcBufs * kTcN)
constexpr int kTcEGWarps = 8;     // two epilogue groups of 4 warps
constexpr int kTcWarps = 16;      // EG0, EG1, {producer, MMA, 2 idle}, samplers: 4 warpgroups
constexpr int kTcSamplerWarp0 = 12;

// ---- tcgen05 / TMEM PTX helpers (sm_100a) -------------------------------------------------
// Shared-memory matrix descriptor, K-major, 128B swizzle (cute UMMA::SmemDescriptor): start
// address >> 4 [0,14), leading byte offset >> 4 [16,30) (unused for swizzled K-major; 1), stride
// byte offset >> 4 [32,46) = 1024 B between 8-row groups, version [46,48) = 1 (sm_100),
// layout type [61,64) = 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// Instruction descriptor, kind::f16 (cute UMMA::InstrDescriptor): c_format F32 [4,6) = 1,
// a/b format [7,10)/[10,13) (F16 = 0, BF16 = 1), K-major A and B, N >> 3 [17,23), M >> 4 [24,29).
template <typename T>
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  constexpr uint32_t f = sizeof(T) == 2 && !std::is_same<T, __half>::value ? 1u : 0u;
  return (1u << 4) | (f << 7) | (f << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// 32 lanes x G columns (fp32) of the warp's TMEM lane quadrant -> G registers per thread
template <int G>
__device__ __forceinline__ void tmem_ld_heads(uint32_t taddr, float (&v)[G]) {
  uint32_t r[G < 2 ? 1 : G];
  if constexpr (G == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
  } else if constexpr (G == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
  } else if constexpr (G == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int g = 0; g < G; ++g) v[g] = __uint_as_float(r[g]);
}

// ---------------------------------------------------------------------------------------
__host__ inline size_t step_tc_score_smem_bytes(int D, int G) {
  const size_t stage = (size_t)(D / 64) * (kTcTileKeys * 128 + kTcN * 128);
  return 1024 + kTcStages * stage + (size_t)2 * 2 * G * 64 * 4 + (size_t)(2 * kTcStages + 2 * kTcBufs) * 8 + 64;
}

template <int N>
__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

template <typename T, int D, int G, int NSW>
__global__ void __launch_bounds__(32 * kTcWarps, 1)
    santa_step_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ,
                         ScoreParams p, SampleParams sp, StepSync sy) {
  static_assert(sizeof(T) == 2 && G <= kTcN, "tensor-core score stage: bf16/fp16, G <= 16");
  static_assert(NSW == 4 && kTcSamplerWarp0 + NSW == kTcWarps, "the sampler group is the last warpgroup");
  constexpr int HALVES = D / 64;
  constexpr int kKBytes = HALVES * kTcTileKeys * 128;  // K tile: [half][128 rows][128 B]
  constexpr int kQBytes = HALVES * kTcN * 128;         // q rows: [half][16 rows][128 B]
  constexpr int kStage = kKBytes + kQBytes;
  constexpr uint32_t kTx = HALVES * (kTcTileKeys * 128 + G * 128);
  constexpr uint32_t kIdesc = umma_idesc_f16<T>(kTcTileKeys, kTcN);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* sSall = reinterpret_cast<float*>(ring + (size_t)kTcStages * kStage);  // [2 EG][2 chunks][G][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(sSall + 2 * 2 * G * 64);
  uint64_t* empty = full + kTcStages;
  uint64_t* tfull = empty + kTcStages;
  uint64_t* tempty = tfull + kTcBufs;
  unsigned char* samp_smem = reinterpret_cast<unsigned char*>(tempty + kTcBufs);
  __shared__ uint32_t sEpoch, sTmem;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
#pragma unroll
    for (int i = 0; i < kTcBufs; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);  // the 4 warps of the epilogue group
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
  // zero the padding rows G..15 of every stage's q block (TMA writes rows 0..G-1 only)
  for (int i = threadIdx.x; i < kTcStages * HALVES * (kTcN - G) * 32; i += blockDim.x) {
    const int w = i % 32, r = G + (i / 32) % (kTcN - G), hs = i / (32 * (kTcN - G));
    reinterpret_cast<uint32_t*>(ring + (size_t)(hs / HALVES) * kStage + kKBytes + (hs % HALVES) * kTcN * 128 +
                                r * 128)[w] = 0u;
  }
  if (warp == kTcEGWarps + 1) tmem_alloc(&sTmem, kTcCols);
  fence_proxy_async_smem();  // the zeroed q rows are read by the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = sTmem;
  const uint32_t epoch = sEpoch;
  const uint32_t tag32 = epoch + 1u, tag16 = epoch % 65535u + 1u;

  const int T2 = (p.Cmax + 1) / 2;           // tiles per unit
  const int total = p.B * p.Hkv * T2;
  const int grid = gridDim.x;
  auto tile_valid = [&](int w, int& unit, int& c2) -> int {  // keys of tile w (<= 0: empty)
    unit = w / T2;
    c2 = w - unit * T2;
    const int b = unit / p.Hkv;
    return min(kTcTileKeys, __ldg(p.seqlens + b) - c2 * kTcTileKeys);
  };

  // per-warpgroup register budgets (each role's code starts with its own setmaxnreg so ptxas
  // allocates it under that budget): 2 x 4 x 112 + 4 x 56 + 4 x 200 = 1920 x 32 <= 64K registers
  if (warp >= kTcEGWarps && warp < kTcSamplerWarp0) setmaxnreg_dec<56>();
  if (warp == kTcEGWarps) {
    // ---------------- TMA producer (one lane) ----------------
    if (lane == 0) {
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmQ);
      const uint64_t pol = l2_policy_evict_first();
      int t = 0;
      for (int w = blockIdx.x; w < total; w += grid) {
        int unit, c2;
        if (tile_valid(w, unit, c2) <= 0) continue;
        const int s = t % kTcStages;
        mbar_wait(&empty[s], ((uint32_t)(t / kTcStages) & 1u) ^ 1u);
        const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
        const int key0 = c2 * kTcTileKeys;
        int32_t row;
        if (p.kv.page_table) {
          const int page = key0 / p.kv.page_size, within = key0 - page * p.kv.page_size;
          const int64_t phys = (int64_t)__ldg(p.kv.page_table + (int64_t)b * p.kv.max_pages + page);
          row = (int32_t)((phys * p.Hkv + kvh) * p.kv.page_size + within);
        } else {
          row = unit * p.kv.page_size + key0;
        }
        unsigned char* st = ring + (size_t)s * kStage;
        mbar_arrive_expect_tx(&full[s], kTx);
#pragma unroll
        for (int h = 0; h < HALVES; ++h) {
          tma_load_2d(st + h * kTcTileKeys * 128, &tmK, 64 * h, row, &full[s], pol);
          tma_load_2d(st + h * kTcTileKeys * 128 + 64 * 128, &tmK, 64 * h, row + 64, &full[s], pol);
          tma_load_2d(st + kKBytes + h * kTcN * 128, &tmQ, 64 * h, b * p.H + kvh * G, &full[s], pol);
        }
        ++t;
      }
      STEP_TRACE(1);
    }
  } else if (warp == kTcEGWarps + 1) {
    // ---------------- MMA issuer (one lane) ----------------
    if (lane == 0) {
      int t = 0;
      for (int w = blockIdx.x; w < total; w += grid) {
        int unit, c2;
        if (tile_valid(w, unit, c2) <= 0) continue;
        const int s = t % kTcStages, bf = t % kTcBufs;
        mbar_wait(&full[s], (uint32_t)(t / kTcStages) & 1u);
        mbar_wait(&tempty[bf], ((uint32_t)(t / kTcBufs) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t st = smem_u32(ring + (size_t)s * kStage);
        const uint32_t tmem_d = tmem_base + (uint32_t)(bf * kTcN);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const int h = kk / 4, off = (kk % 4) * 32;
          umma_f16(tmem_d, umma_desc_sw128(st + h * kTcTileKeys * 128 + off),
                   umma_desc_sw128(st + kKBytes + h * kTcN * 128 + off), kIdesc, kk > 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);  // the stage is free once these MMAs have read it
        umma_commit(&tfull[bf]);  // the accumulator is ready
        ++t;
      }
    }
    __syncwarp();
  } else if (warp < kTcEGWarps) {
    // ---------------- epilogue groups ----------------
    setmaxnreg_dec<112>();
    const int e = warp >> 2, wq = warp & 3;
    float* sS = sSall + (size_t)e * 2 * G * 64;
    int t = 0;
    int cur_unit = -1;
    for (int w = blockIdx.x; w < total; w += grid) {
      int unit, c2;
      const int n_valid = tile_valid(w, unit, c2);
      if (n_valid <= 0) continue;
      if ((t & 1) != e) {
        ++t;
        continue;
      }
      (void)cur_unit;
      const int bf = t % kTcBufs;
      mbar_wait(&tfull[bf], (uint32_t)(t / kTcBufs) & 1u);
      tc_fence_after();
      float v[G];
      tmem_ld_heads<G>(tmem_base + ((uint32_t)(32 * wq) << 16) + (uint32_t)(bf * kTcN), v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[bf]);
      const int key = 32 * wq + lane;  // key within the tile: chunk key >> 6, position key & 63
#pragma unroll
      for (int g = 0; g < G; ++g)
        sS[((key >> 6) * G + g) * 64 + (key & 63)] = key < n_valid ? v[g] * p.scale_log2 : -INFINITY;
      named_bar_sync(2 + e, 128);
      if (wq < 2) {
        const int nv = min(64, n_valid - 64 * wq);
        if (nv > 0) {
          const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
          const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
          const int c = 2 * c2 + wq;
          warp_chunk_epilogue_ll<G>(sS + wq * G * 64, nv, sy.stash + (bh0 * p.Cmax + c) * 64,
                                    sy.rec + bh0 * p.Cmax + c, p.Cmax, tag32, tag16);
        }
      }
      named_bar_sync(2 + e, 128);  // sS is rewritten by the group's next tile
      ++t;
    }
    if (lane == 0 && sy.trace) STEP_TRACE(2 + warp);
  } else if (warp >= kTcSamplerWarp0) {
    // ---------------- sampler group ----------------
    setmaxnreg_inc<200>();
    step_sampler_loop<T, D, G, NSW>(sp, sy, samp_smem, tag32, tag16);
  }
  // ---------------- teardown: TMEM, then the exit ticket (the last CTA out advances the epoch) ----
  tc_fence_before();
  __syncthreads();
  if (warp == kTcEGWarps + 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTcCols);
  }
  if (threadIdx.x == 0) {
    if (atomicAdd(sy.exit_ticket, 1u) == (uint32_t)(grid - 1)) {
      *sy.exit_ticket = 0u;
      *sy.epoch = epoch + 1u;
    }
  }
}

}  // namespace santa
