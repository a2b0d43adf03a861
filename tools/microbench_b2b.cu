// microbench_b2b.cu -- BACK-TO-BACK streaming throughput of a 64 MiB (config-2 K) read, the
// regime bench.py times (consecutive launches over rotating buffers > L2, events around the
// whole loop).  Tools only, not part of libsanta.  Questions it answers:
//   * per-launch floor of an empty persistent grid (launch + drain cost when back-to-back)
//   * TMA ring (1 producer lane, NC consumer warps that only wait+release) vs plain LDG.128
//     streams at several occupancies vs 1-D bulk copies, for block-contiguous and chunk-
//     interleaved (CTA i takes 16 KiB chunks i, i+grid, ...) orderings
//   * a per-CTA %globaltimer trace (start, first byte, last byte, end) of one launch
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_b2b tools/microbench_b2b.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../paper_2605_01910_b200/csrc/tma.cuh"

using namespace santa;

__device__ __forceinline__ uint4 ldg_stream_(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__global__ void empty_kernel() {}

// ring: MODE 0 = 2-D TMA (2 boxes of 64 rows x 128 B per 16 KiB stage), 1 = 1-D bulk.
// ORDER 0 = block-contiguous stage ranges, 1 = interleaved (stage s -> CTA s % grid).
template <int MODE, int ORDER>
__global__ void __launch_bounds__(32 * 9, 1) ring_kernel(const __grid_constant__ CUtensorMap tm, const char* base,
                                                        int nst_total, int spw, int ncons,
                                                        unsigned long long* sink, unsigned long long* trace) {
  constexpr int SB = 16384;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nsl = spw * ncons;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)nsl * SB);
  uint64_t* empty = full + nsl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) {
    t0 = gt();
    for (int i = 0; i < nsl; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  int lo, cnt, step;
  if (ORDER == 0) {
    lo = (int)((long long)nst_total * blockIdx.x / gridDim.x);
    cnt = (int)((long long)nst_total * (blockIdx.x + 1) / gridDim.x) - lo;
    step = 1;
  } else {
    lo = blockIdx.x;
    cnt = nst_total > (int)blockIdx.x ? (nst_total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    step = gridDim.x;
  }
  if (warp == ncons) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      for (int k = 0; k < cnt; ++k) {
        const int w = k % ncons, i = k / ncons;
        const int slot = w * spw + i % spw, ph = (i / spw) & 1;
        mbar_wait(&empty[slot], ph ^ 1);
        const long long s = lo + (long long)k * step;
        mbar_arrive_expect_tx(&full[slot], SB);
        if (MODE == 0) {
          tma_load_2d(ring + slot * SB, &tm, 0, (int)(s * 64), &full[slot], pol);
          tma_load_2d(ring + slot * SB + SB / 2, &tm, 64, (int)(s * 64), &full[slot], pol);
        } else {
          bulk_load(ring + slot * SB, base + s * SB, SB, &full[slot], pol);
        }
      }
    }
    return;
  }
  if (warp >= ncons) return;
  unsigned long long acc = 0, tfirst = 0, tlast = 0;
  int i = 0;
  for (int k = warp; k < cnt; k += ncons, ++i) {
    const int slot = warp * spw + i % spw, ph = (i / spw) & 1;
    mbar_wait(&full[slot], ph);
    if (trace && lane == 0) {
      if (!tfirst) tfirst = gt();
      tlast = gt();
    }
    acc += *reinterpret_cast<const unsigned int*>(ring + slot * SB + lane * 4);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 0x123456789ull) sink[0] = acc;
  if (trace && lane == 0) {
    unsigned long long* tr = trace + (size_t)blockIdx.x * 4 * 8 + warp * 4;
    tr[1] = tfirst;
    tr[2] = tlast;
    tr[3] = gt();
    if (warp == 0) tr[0] = t0;
  }
}

// plain LDG.128 stream, U loads in flight per thread.  ORDER 0: block-contiguous; 1: 16 KiB
// chunks interleaved over blocks.
template <int ORDER>
__global__ void ldg_kernel(const uint4* __restrict__ p, long long n16, unsigned long long* sink) {
  unsigned long long acc = 0;
  constexpr int U = 8;
  if (ORDER == 0) {
    const long long per = (n16 + gridDim.x - 1) / gridDim.x;
    const long long lo = blockIdx.x * per, hi = min(n16, lo + per);
    for (long long i = lo + threadIdx.x; i < hi; i += U * blockDim.x) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = i + u * blockDim.x;
        v[u] = j < hi ? ldg_stream_(p + j) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
    }
  } else {
    // chunk = 1024 uint4 = 16 KiB; a block of 512 threads reads 2 uint4 per thread per chunk;
    // U/2 chunks in flight
    const long long nch = n16 / 1024;
    for (long long c = blockIdx.x; c < nch; c += (long long)gridDim.x * (U / 2)) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long cc = c + (long long)(u / 2) * gridDim.x;
        v[u] = cc < nch ? ldg_stream_(p + cc * 1024 + (u & 1) * 512 + threadIdx.x) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
    }
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

int main() {
  const size_t bytes = 64ull << 20;
  const int NB = 8;  // 8 x 64 MiB = 512 MiB rotated (> 4x L2)
  char* K;
  cudaMalloc(&K, bytes * NB);
  cudaMemset(K, 1, bytes * NB);
  unsigned long long *sink, *trace;
  cudaMalloc(&sink, 8);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&trace, (size_t)nsm * 32 * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  std::vector<CUtensorMap> tms(NB);
  for (int b = 0; b < NB; ++b) {
    cuuint64_t dims[2] = {128, (cuuint64_t)(bytes / 256)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    enc(&tms[b], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K + b * bytes, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ITER = 64;
  auto b2b = [&](auto&& fn, const char* name, size_t nbytes) {
    for (int i = 0; i < 8; ++i) fn(i);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < ITER; ++i) fn(i);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / ITER;
    printf("%-60s %8.2f us/launch  %7.0f GB/s  (%s)\n", name, us, nbytes ? nbytes / (us * 1e-6) / 1e9 : 0.0,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  };
  b2b([&](int) { empty_kernel<<<nsm, 32>>>(); }, "empty kernel, grid SMs x 32", 0);
  b2b([&](int) { empty_kernel<<<nsm, 288>>>(); }, "empty kernel, grid SMs x 288", 0);
  const int nst = (int)(bytes / 16384);
  for (int ncons : {4, 6, 8})
    for (int spw : {2, 3}) {
      const size_t smem = 1024 + (size_t)spw * ncons * 16384 + 2 * spw * ncons * 8;
      if (smem > 227 * 1024) continue;
      for (int order = 0; order < 2; ++order)
        for (int mode = 0; mode < 2; ++mode) {
          auto kern = mode == 0 ? (order ? ring_kernel<0, 1> : ring_kernel<0, 0>)
                                : (order ? ring_kernel<1, 1> : ring_kernel<1, 0>);
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          char name[128];
          snprintf(name, sizeof name, "%s %s ring %d cons x %d slots", mode ? "bulk-1D" : "TMA-2D ",
                   order ? "interleaved" : "contiguous ", ncons, spw);
          b2b([&](int i) {
                kern<<<nsm, 32 * (ncons + 1), smem>>>(tms[i % NB], K + (i % NB) * bytes, nst, spw, ncons, sink,
                                                        nullptr);
              },
              name, bytes);
        }
    }
  for (int occ : {1, 2, 4, 8})
    for (int order = 0; order < 2; ++order) {
      char name[128];
      snprintf(name, sizeof name, "LDG.128 x8 %s grid %d x 512", order ? "interleaved" : "contiguous ", nsm * occ);
      auto kern = order ? ldg_kernel<1> : ldg_kernel<0>;
      b2b([&](int i) { kern<<<nsm * occ, 512>>>((const uint4*)(K + (i % NB) * bytes), bytes / 16, sink); }, name,
          bytes);
    }
  // one traced launch (TMA-2D contiguous, 6 x 2) in the middle of a back-to-back sequence
  {
    const int ncons = 6, spw = 2;
    const size_t smem = 1024 + (size_t)spw * ncons * 16384 + 2 * spw * ncons * 8;
    for (int order = 0; order < 2; ++order) {
      auto kern = order ? ring_kernel<0, 1> : ring_kernel<0, 0>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaMemset(trace, 0, (size_t)nsm * 32 * 8);
      for (int i = 0; i < 6; ++i)
        kern<<<nsm, 32 * (ncons + 1), smem>>>(tms[i % NB], K, nst, spw, ncons, sink, i == 4 ? trace : nullptr);
      cudaDeviceSynchronize();
      std::vector<unsigned long long> tr((size_t)nsm * 32);
      cudaMemcpy(tr.data(), trace, tr.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, tend = 0;
      std::vector<double> start, first, last, end;
      for (int b = 0; b < nsm; ++b) t0 = std::min(t0, tr[(size_t)b * 32]);
      for (int b = 0; b < nsm; ++b) {
        unsigned long long f = ~0ull, l = 0, e = 0;
        for (int w = 0; w < ncons; ++w) {
          const unsigned long long* x = &tr[(size_t)b * 32 + w * 4];
          if (x[1]) f = std::min(f, x[1]);
          l = std::max(l, x[2]);
          e = std::max(e, x[3]);
        }
        start.push_back((tr[(size_t)b * 32] - t0) * 1e-3);
        first.push_back((f - t0) * 1e-3);
        last.push_back((l - t0) * 1e-3);
        end.push_back((e - t0) * 1e-3);
        tend = std::max(tend, e);
      }
      auto stat = [](std::vector<double> v, const char* n) {
        std::sort(v.begin(), v.end());
        printf("   %-22s min %6.2f  p50 %6.2f  max %6.2f us\n", n, v.front(), v[v.size() / 2], v.back());
      };
      printf("trace (TMA-2D %s 6x2, one launch in a back-to-back run; t=0 at first CTA start):\n",
             order ? "interleaved" : "contiguous");
      stat(start, "CTA start");
      stat(first, "first stage landed");
      stat(last, "last stage landed");
      stat(end, "CTA end");
    }
  }
  return 0;
}
