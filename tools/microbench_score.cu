// microbench_score.cu -- tunes the streaming score kernel (tools only, not part of libsanta).
// Config-2 shape: B=1, H=32, H_kv=8, d=128, bf16, n=32768, L=64.  Each variant is launched
// back-to-back over 4 rotating KV caches (512 MiB > 4x L2), timed with CUDA events.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2605_01910_b200/csrc \
//        -o tools/microbench_score tools/microbench_score.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "score_kernels.cuh"

using namespace santa;
using bf16 = __nv_bfloat16;

__global__ void fill_kernel(bf16* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = __float2bfloat16(((x & 0xffff) / 65536.0f - 0.5f) * 3.4f);
  }
}

int main() {
  const int B = 1, H = 32, Hkv = 8, D = 128, n = 32768, L = 64, NR = 4;
  const int Cmax = n / L;
  const size_t kelems = (size_t)B * Hkv * n * D;
  std::vector<bf16*> Ks(NR), qs(NR);
  for (int r = 0; r < NR; ++r) {
    cudaMalloc(&Ks[r], kelems * 2);
    cudaMalloc(&qs[r], (size_t)B * H * D * 2);
    fill_kernel<<<1024, 256>>>(Ks[r], kelems, 17 + r);
    fill_kernel<<<8, 256>>>(qs[r], (size_t)B * H * D, 99 + r);
  }
  int* seqlens;
  cudaMalloc(&seqlens, 4);
  cudaMemcpy(seqlens, &n, 4, cudaMemcpyHostToDevice);
  float* stash;
  float2* cstats;
  uint32_t* misc;
  cudaMalloc(&stash, (size_t)B * H * Cmax * L * 4);
  cudaMalloc(&cstats, (size_t)B * H * Cmax * 8);
  cudaMalloc(&misc, 4096);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  std::vector<CUtensorMap> tms(NR);
  for (int r = 0; r < NR; ++r) {
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)B * Hkv * n};
    cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    enc(&tms[r], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Ks[r], dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  auto params = [&](int r) {
    ScoreParams p{};
    p.q = qs[r];
    p.K = Ks[r];
    p.kv.page_table = nullptr;
    p.kv.page_size = n;
    p.kv.max_pages = 1;
    p.kv.n_kv_heads = Hkv;
    p.seqlens = seqlens;
    p.B = B; p.H = H; p.Hkv = Hkv;
    p.scale_log2 = 0.08838834764f * 1.4426950408889634f;
    p.stash = stash; p.cstats = cstats; p.Cmax = Cmax; p.L = L; p.stash_stride = Cmax * L;
    p.tickets = misc; p.flags = misc + 64;
    return p;
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, int nw, int spw, const char* name) {
    const size_t smem = 1024 + (size_t)nw * 4 * L * 4 + (size_t)nw * spw * (16384 + 16);
    if (smem > 227 * 1024) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int K = 40;
    for (int i = 0; i < 8; ++i) kern<<<nsm, 32 * (nw + 1), smem>>>(tms[i % NR], params(i % NR));
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < K; ++i) kern<<<nsm, 32 * (nw + 1), smem>>>(tms[i % NR], params(i % NR));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / K;
    printf("%-28s smem %6zu  %7.2f us/launch  %7.0f GB/s  (%s)\n", name, smem, us, kelems * 2 / (us * 1e-6) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  };
#define V(NW, SPW, A) run(score_stream_kernel<bf16, 128, 4, NW, SPW, A>, NW, SPW, "score_stream NW=" #NW " SPW=" #SPW " ablate=" #A)
  for (int rep = 0; rep < 2; ++rep) {
    V(2, 6, 0); V(2, 6, 1); V(2, 6, 2);
    V(4, 2, 0); V(4, 2, 1); V(4, 2, 2);
    V(6, 2, 0); V(6, 2, 1); V(6, 2, 2);
    V(8, 1, 0); V(8, 1, 1); V(8, 1, 2);
  }
  return 0;
}
