// microbench_stream.cu -- isolates HBM streaming throughput of the load mechanisms the score
// pass can use (tools only, not part of libsanta):
//   A: 2-D TMA ring (64x64 bf16 boxes, 128B swizzle), 1 producer lane, NC consumer warps that
//      only wait + release (no math)
//   B: 1-D cp.async.bulk ring (contiguous 16 KiB stages), same consumers
//   C: plain 128-bit LDG stream (unrolled), grid = SMs x occ
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o microbench_stream tools/microbench_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "../paper_2605_01910_b200/csrc/tma.cuh"

__device__ __forceinline__ uint4 ldg_stream_(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

using namespace santa;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int MODE>  // 0 = 2-D TMA, 1 = 1-D bulk
__global__ void __launch_bounds__(32 * 9, 1) ring_kernel(const __grid_constant__ CUtensorMap tm, const char* base,
                                                        int nstages_total, int spw, int nconsumers, int stage_bytes,
                                                        unsigned long long* sink) {
  // consumer warp w owns slots [w*spw, (w+1)*spw): its i-th stage uses slot w*spw + i % spw,
  // parity (i / spw) & 1 -- a slot is only ever reused by its own warp, in order.
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nst = spw * nconsumers;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)nst * stage_bytes);
  uint64_t* empty = full + nst;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int mine = nstages_total > (int)blockIdx.x ? (nstages_total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (warp == nconsumers) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      for (int k = 0; k < mine; ++k) {
        const int w = k % nconsumers, i = k / nconsumers;
        const int slot = w * spw + i % spw, ph = (i / spw) & 1;
        mbar_wait(&empty[slot], ph ^ 1);
        const long long s = blockIdx.x + (long long)k * gridDim.x;
        mbar_arrive_expect_tx(&full[slot], stage_bytes);
        if (MODE == 0) {
          const int rows_per_stage = stage_bytes / 256;  // 128 bf16 per row (2 boxes of rows x 64)
          tma_load_2d(ring + slot * stage_bytes, &tm, 0, (int)(s * rows_per_stage), &full[slot], pol);
          tma_load_2d(ring + slot * stage_bytes + stage_bytes / 2, &tm, 64, (int)(s * rows_per_stage), &full[slot],
                      pol);
        } else {
          bulk_load(ring + slot * stage_bytes, base + s * stage_bytes, stage_bytes, &full[slot]);
        }
      }
    }
    return;
  }
  if (warp >= nconsumers) return;
  unsigned long long acc = 0;
  int i = 0;
  for (int k = warp; k < mine; k += nconsumers, ++i) {
    const int slot = warp * spw + i % spw, ph = (i / spw) & 1;
    mbar_wait(&full[slot], ph);
    acc += *reinterpret_cast<const unsigned int*>(ring + slot * stage_bytes + lane * 4);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

__global__ void ldg_kernel(const uint4* __restrict__ p, long long n16, unsigned long long* sink) {
  // block-contiguous: block b reads [b*per, (b+1)*per), U loads in flight per thread
  unsigned long long acc = 0;
  const long long per = (n16 + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(n16, lo + per);
  constexpr int U = 8;
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
  if (acc == 0x123456789ull) sink[0] = acc;
}
__global__ void empty_kernel() {}

int main() {
  const size_t maxbytes = 2048ull << 20;
  char* K;
  cudaMalloc(&K, maxbytes);
  cudaMemset(K, 1, maxbytes);
  char* flush;
  const size_t fbytes = 512ull << 20;
  cudaMalloc(&flush, fbytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  size_t bytes = 0;
  char* rflush;
  cudaMalloc(&rflush, 256ull << 20);
  cudaMemset(rflush, 0, 256ull << 20);
  int clean = 0;
  auto timeit = [&](auto&& fn, const char* name) {
    float best = 1e9, sum = 0;
    for (int it = 0; it < 12; ++it) {
      cudaMemsetAsync(flush, it, fbytes);
      if (clean) ldg_kernel<<<nsm * 4, 512>>>((const uint4*)rflush, (256ull << 20) / 16, sink);
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) {
        best = ms < best ? ms : best;
        sum += ms;
      }
    }
    const cudaError_t err = cudaGetLastError();
    printf("%-64s best %8.2f us  mean %8.2f us  -> %7.0f GB/s  (%s)\n", name, best * 1e3, sum / 10 * 1e3,
           bytes / (best * 1e-3) / 1e9, cudaGetErrorString(err));
    fflush(stdout);
  };
  for (clean = 0; clean < 2; ++clean) {
  printf("==== flush: 512 MiB write%s ====\n", clean ? " + 256 MiB read (L2 left clean)" : " only (L2 left dirty)");
  bytes = 0;
  timeit([&] { empty_kernel<<<nsm, 32>>>(); }, "empty kernel (event overhead)");
  for (size_t mb : {16, 64, 256}) {
    bytes = mb << 20;
    const int rows = bytes / 256;
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode = 0; mode < 2; ++mode) {
      const int sb = 16384, ncons = 4, spw = 3;
      const size_t smem = 1024 + (size_t)spw * ncons * sb + 2 * spw * ncons * 8;
      auto kern = mode == 0 ? ring_kernel<0> : ring_kernel<1>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      char name[128];
      snprintf(name, sizeof name, "%5zu MiB %s 16KiB x 4 cons x 3 slots", mb, mode == 0 ? "TMA-2D " : "bulk-1D");
      timeit([&] { kern<<<nsm, 32 * (ncons + 1), smem>>>(tm, K, (int)(bytes / sb), spw, ncons, sb, sink); }, name);
    }
    for (int occ : {2, 4, 8}) {
      char name[128];
      snprintf(name, sizeof name, "%5zu MiB LDG.128 x8 grid %d x 512", mb, nsm * occ);
      timeit([&] { ldg_kernel<<<nsm * occ, 512>>>((const uint4*)K, bytes / 16, sink); }, name);
    }
  }
  }
  return 0;
}
