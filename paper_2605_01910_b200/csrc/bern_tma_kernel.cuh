// bern_tma_kernel.cuh -- the Bernoulli score stage (Eq. 5, Eq. 6
// P:486-495) for decode on bf16 feature-major caches, as a persistent TMA stream on the tensor pipe.
//
// p_hat_g[k] = sum_{i in F} w_{g,i} Kt[i][k] is a contraction over the selected features F of the
// unit (b, kv-head): with the keys as M, the selected features as K and the G heads as N it is an
// [n x |F|] x [|F| x G] product, exactly the exact score pass's shape with K^T instead of K.  So:
//   * producer warp: per work item (unit, 1024-key block) and per group of 16 selected features, one
//     ring stage = 16 row segments of 2 KB (one cp.async.bulk per row, the features' ids from the
//     compacted selection list) + the group's 768 B of B fragments; rows at a 2064-B pitch (a 16-B
//     skew per row: the 8 rows of an ldmatrix tile hit 8 distinct 4-bank groups).  Rows past |F|
//     repeat the last selected row (weight 0; an L2 hit).  2-KB copies: with 512-B copies (256-key
//     items) the stream reached 2.3 TB/s -- a bulk copy is issued through the uniform datapath one
//     lane at a time (ELECT / R2UR / UBLKCP loop), ~60 cycles per request per SM.
//   * 8 consumer warps, 128 keys (two 64-key chunks) each: per stage and 16-key tile one
//     ldmatrix.x4.trans (the K^T tile
//     arrives key-major = the A fragment of m16n8k16) and three mma.sync, one per bf16 PART of the
//     weights: w = w_hi + w_mid + w_lo (each bf16, w_hi = rn(w), w_mid = rn(w - w_hi), w_lo =
//     rn(w - w_hi - w_mid): |w - sum| <= 2^-24 |w|, i.e. the fp32 weights to their last bit), fp32
//     accumulation, the parts summed (lo + mid) + hi in the epilogue.  Then the exact pass's L = 64
//     register epilogue -> the sampler's stash / chunk stats (sub64 layout), unchanged downstream.
// The B fragments come from bern_weights_kernel (p.wfrag: [unit][|F|/16 groups][3 parts][32 lanes]
// uint2), built once per unit.  The FMA stream it replaces (bern_stream_kernel) issued ~45
// instructions per 16-B row segment per lane (address arithmetic, bf16 unpacking, 16 FFMA2) and was
// issue/latency bound at 0.6 of peak; here a 512-B row costs the consumers ~1 instruction.
#pragma once
#include "bernoulli_kernels.cuh"
#include "dense_stream_kernel.cuh"

namespace santa {

constexpr int kBtWarps = 8;                          // consumer warps
constexpr int kBtWarpKeys = 128;                     // keys per consumer warp (two 64-key chunks)
constexpr int kBtTiles = kBtWarpKeys / 16;           // m16 tiles per warp
constexpr int kBtKeys = kBtWarpKeys * kBtWarps;      // 1024 keys per work item
constexpr int kBtRows = 16;                          // feature rows per stage (the MMA K)
constexpr int kBtPitch = kBtKeys * 2 + 16;           // 2064 B row pitch (bank skew)
constexpr int kBtFragBytes = 3 * 32 * 8;             // B fragments of one 16-feature group
constexpr int kBtStageBytes = kBtRows * kBtPitch + kBtFragBytes;  // 33792 B
constexpr int kBtSlots = 6;                          // ring depth (one CTA per SM: 192 KB in flight)
constexpr int kBtProducers = 4;                      // producer warps (rows split between them)
constexpr int kBtMinPage = 64;                       // paged pools: P % 1024 == 0 or 1024 % P == 0, P >= 64

__host__ __device__ constexpr size_t bern_tma_smem_bytes(int G) {
  return 128 + (size_t)kBtSlots * kBtStageBytes + (size_t)kBtWarps * G * 64 * 4 + 2 * kBtSlots * 8;
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Producer-side per-item metadata (loaded one item ahead).
template <int D>
struct BtMeta {
  int seqlen, nsel;
  int sel[D / 32];  // lane l: sel[l + 32 r]
  int64_t base;     // element offset of feature 0's row segment (contiguous / one page per block)
};

template <typename T, int D, int G>
__global__ void __launch_bounds__(32 * (kBtWarps + kBtProducers), 1) bern_tma_kernel(BernParams p, int items) {
  static_assert(sizeof(T) == 2, "16-bit caches");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  float* sSall = reinterpret_cast<float*>(ring + (size_t)kBtSlots * kBtStageBytes);  // [NW][G][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(sSall + kBtWarps * G * 64);
  uint64_t* empty = full + kBtSlots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBtSlots; ++i) {
      mbar_init(&full[i], kBtProducers);
      mbar_init(&empty[i], kBtWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait_primary();  // the weights kernel's selection, weights and fragments
  pdl_launch_dependents();
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.flags) *p.flags = 0u;
  const int nblk = (p.score_stride + kBtKeys - 1) / kBtKeys;
  const int P = p.page_table ? p.page_size : p.score_stride;  // row length of the feature-major layout

  if (warp >= kBtWarps) {
    // ---------------- producers: warp pw issues rows [pw 16/NP, (pw + 1) 16/NP) of every stage ----------------
    constexpr int kRowsPer = kBtRows / kBtProducers;
    const int pw = warp - kBtWarps;
    const T* Kt = reinterpret_cast<const T*>(p.Kt);
    const uint64_t pol = l2_policy_evict_first();
    // a paged pool with P < 1024 (host: 1024 % P == 0): one copy per row and page ("piece")
    const int npc = (p.page_table != nullptr && P < kBtKeys) ? kBtKeys / P : 1;
    const int pk = npc > 1 ? P : kBtKeys;  // keys per piece
    auto load_meta = [&](int it, BtMeta<D>& m) {
      m.seqlen = 0;
      m.nsel = 0;
      if (it >= items) return;
      const int unit = it / nblk, blk = it - unit * nblk;
      const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
      const int k0 = blk * kBtKeys;
      m.seqlen = __ldg(p.seqlens + b);
      m.nsel = __ldcg(p.sel_n + unit);
#pragma unroll
      for (int r = 0; r < D / 32; ++r) m.sel[r] = __ldcg(p.sel + (size_t)unit * D + lane + 32 * r);
      const int page = k0 / P, within = k0 - page * P;
      const int64_t phys =
          p.page_table ? (page < p.max_pages ? (int64_t)__ldg(p.page_table + (int64_t)b * p.max_pages + page) : 0) : b;
      m.base = ((phys * p.Hkv + kvh) * D) * (int64_t)P + within;
    };
    BtMeta<D> cur, nxt;
    load_meta(blockIdx.x, nxt);
    int k = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      cur = nxt;
      load_meta(it + gridDim.x, nxt);  // in flight while this item's copies are issued
      const int unit = it / nblk, blk = it - unit * nblk;
      const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
      const int k0 = blk * kBtKeys;
      if (k0 >= cur.seqlen) continue;
      const int ng = (cur.nsel + kBtRows - 1) / kBtRows;
      // bytes of piece pc of every row: its keys up to the sequence end, rounded up to 8 keys = 16 B
      // (inside the row / page: P % 8 == 0, host-checked); 0 past the end
      uint32_t tx = 0;
      for (int pc = 0; pc < npc; ++pc) tx += 2u * (uint32_t)max(0, min(pk, (cur.seqlen - k0 - pc * pk + 7) & ~7));
      const uint2* frag = p.wfrag + (size_t)unit * (D / 16) * 96;
      for (int kg = 0; kg < ng; ++kg, ++k) {
        const int slot = k % kBtSlots;
        mbar_wait(&empty[slot], ((uint32_t)(k / kBtSlots) & 1u) ^ 1u);
        if (lane == 0) mbar_arrive_expect_tx(&full[slot], kRowsPer * tx + (pw == 0 ? kBtFragBytes : 0));
        __syncwarp();
        const uint32_t stage = smem_u32(ring + (size_t)slot * kBtStageBytes);
        if (lane == 0 && pw == 0)  // the fragments are re-read by every item of the unit: no evict-first hint
          bulk_g2s(stage + kBtRows * kBtPitch, frag + (size_t)kg * 96, kBtFragBytes, &full[slot]);
        for (int e0 = 0; e0 < kRowsPer * npc; e0 += 32) {  // copy e = (row e / npc, piece e % npc)
          const int e = e0 + lane;
          const int row = kRowsPer * pw + e / npc, pc = e % npc;
          const int s = min(kBtRows * kg + row, cur.nsel - 1);  // rows past |F| repeat the last one (weight 0)
          int f = 0;  // selection entry s lives in lane s % 32, register s / 32
#pragma unroll
          for (int r = 0; r < D / 32; ++r) {
            const int v = __shfl_sync(0xffffffffu, cur.sel[r], s & 31);
            if ((s >> 5) == r) f = v;
          }
          const int nkp = min(pk, (cur.seqlen - k0 - pc * pk + 7) & ~7);
          if (e < kRowsPer * npc && nkp > 0) {
            int64_t base = cur.base;
            if (npc > 1) {  // page of this piece (small-page pools only)
              const int page = (k0 + pc * pk) / P;
              const int64_t phys = (int64_t)__ldg(p.page_table + (int64_t)b * p.max_pages + page);
              base = ((phys * p.Hkv + kvh) * D) * (int64_t)P;
            }
            bulk_g2s(stage + row * kBtPitch + pc * pk * 2, Kt + base + (int64_t)f * P, 2u * (uint32_t)nkp,
                     &full[slot], pol);
          }
        }
      }
    }
  } else {
    // ---------------- consumers: warp w owns keys [128 w, 128 w + 128) of every item ----------------
    float* sS = sSall + warp * G * 64;
    const float sl2 = p.scale * kLog2e;
    const int j = lane >> 3, r8 = lane & 7;
    // ldmatrix.x4.trans source row of this lane: feature row r8 + 8 (j / 2), keys 128 w + 8 (j % 2) + 16 t
    const uint32_t a_off = (uint32_t)((r8 + 8 * (j >> 1)) * kBtPitch + (kBtWarpKeys * warp + 8 * (j & 1)) * 2);
    int k = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int unit = it / nblk, blk = it - unit * nblk;
      const int b = unit / p.Hkv, kvh = unit - b * p.Hkv;
      const size_t bh0 = (size_t)b * p.H + (size_t)kvh * G;
      const int seqlen = __ldg(p.seqlens + b);
      const int wk0 = blk * kBtKeys + kBtWarpKeys * warp;  // this warp's first key
      if (blk * kBtKeys >= seqlen) {  // block past the sequence: no stage was issued
#pragma unroll
        for (int h = 0; h < kBtWarpKeys / 64; ++h) {
          const int c = wk0 / 64 + h;
          if (lane < G && c < p.Cmax) p.cstats[(bh0 + lane) * p.Cmax + c] = make_float2(-INFINITY, 0.f);
        }
        continue;
      }
      const int ng = (__ldcg(p.sel_n + unit) + kBtRows - 1) / kBtRows;
      float acc[3][kBtTiles][4];
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int t = 0; t < kBtTiles; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[q][t][e] = 0.f;
      for (int kg = 0; kg < ng; ++kg, ++k) {
        const int slot = k % kBtSlots;
        mbar_wait(&full[slot], (uint32_t)(k / kBtSlots) & 1u);
        const uint32_t stage = smem_u32(ring + (size_t)slot * kBtStageBytes);
        uint2 bf[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const uint32_t ad = stage + kBtRows * kBtPitch + q * 256 + lane * 8;
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(bf[q].x), "=r"(bf[q].y) : "r"(ad));
        }
        uint32_t a[kBtTiles][4];
#pragma unroll
        for (int t = 0; t < kBtTiles; ++t) ldsm_x4_trans(stage + a_off + 32 * t, a[t][0], a[t][1], a[t][2], a[t][3]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
#pragma unroll
        for (int t = 0; t < kBtTiles; ++t)
#pragma unroll
          for (int q = 0; q < 3; ++q) Mma<T>::run(acc[q][t], a[t][0], a[t][1], a[t][2], a[t][3], bf[q].x, bf[q].y);
      }
#pragma unroll
      for (int h = 0; h < kBtWarpKeys / 64; ++h) {
        const int chunk_start = wk0 + 64 * h, c = chunk_start / 64;
        const int n_valid = min(64, seqlen - chunk_start);
        if (n_valid <= 0) {
          if (lane < G && c < p.Cmax) p.cstats[(bh0 + lane) * p.Cmax + c] = make_float2(-INFINITY, 0.f);
          continue;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float sum[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) sum[e] = (acc[2][4 * h + t][e] + acc[1][4 * h + t][e]) + acc[0][4 * h + t][e];
          store_tile_scores<G>(sS, 64, 16 * t, n_valid, sum, sl2);
        }
        __syncwarp();
        warp_chunk_epilogue<G>(sS, 64, n_valid, p.stash + bh0 * p.stash_stride + chunk_start, p.stash_stride,
                               p.cstats + bh0 * p.Cmax + c, p.Cmax);
        __syncwarp();
      }
    }
  }
}

}  // namespace santa
