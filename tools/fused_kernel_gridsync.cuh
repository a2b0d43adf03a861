// fused_kernel_gridsync.cuh -- (tools only) the earlier single-launch step with grid.sync(), kept
// for comparison in microbench_sample; superseded by csrc/step_kernel.cuh (per-unit counters).
//
// Cooperative launch, one CTA per SM (co-residency guaranteed):
//   phase 1  score_stream_body: TMA ring + mma.sync score pass, chunk stats + prefix stash
//   grid.sync()                 -- the global dependency of sampling ("requires a global CDF")
//   phase 2  work items (b, h, split) over the CTAs: sample_item (thresholds, fp64 chunk CDF,
//            inverse CDF, gather-add) reusing the ring's shared memory
//   grid.sync(), then a fixed-order sum of the split partials (deterministic) -> out
// Replaces the score kernel + sampler kernel pair (one launch and the inter-kernel gap saved).
#pragma once
#include <cooperative_groups.h>

#include "../paper_2605_01910_b200/csrc/sample_kernels.cuh"
#include "../paper_2605_01910_b200/csrc/score_kernels.cuh"

namespace santa {

template <typename T, int D, int G, int NW, int SPW>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    santa_fused_kernel(const __grid_constant__ CUtensorMap tmK, ScoreParams sp, SampleParams pp) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  namespace cg = cooperative_groups;
  unsigned long long* tr = pp.trace ? pp.trace + (size_t)pp.B * pp.H * 16 + blockIdx.x * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();
  score_stream_body<T, D, G, NW, SPW>(&tmK, sp, smem_raw);
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[1] = gtimer();
  cg::grid_group grid = cg::this_grid();
  grid.sync();
  if (tr && threadIdx.x == 0) tr[2] = gtimer();
  const int CS = pp.cluster;
  const int items = pp.B * pp.H * CS;
  const float invS = 1.0f / (float)pp.S;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int rank = it % CS, bh = it / CS;
    const int b = bh / pp.H, h = bh - b * pp.H;
    const float* sPart = sample_item<T, D, G>(pp, b, h, rank, CS, smem_raw);
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      if (CS == 1) store_out<T, D>(pp, (size_t)bh, d, sPart[d] * invS);
      else pp.split_partial[(size_t)it * D + d] = sPart[d];
    }
    __syncthreads();  // sPart is rewritten by the next item
  }
  if (tr && threadIdx.x == 0) tr[3] = gtimer();
  if (CS > 1) {
    grid.sync();
    if (tr && threadIdx.x == 0) tr[4] = gtimer();
    for (int bh = blockIdx.x; bh < pp.B * pp.H; bh += gridDim.x)
      for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float s = 0.f;
        for (int r = 0; r < CS; ++r) s += __ldcg(pp.split_partial + ((size_t)bh * CS + r) * D + d);
        store_out<T, D>(pp, (size_t)bh, d, s * invS);
      }
  }
  if (tr && threadIdx.x == 0) tr[5] = gtimer();
}

}  // namespace santa
