// microbench_fast.cu -- timeline of the low-latency sampler (sample_fast.cuh) behind the streaming
// score pass at config 2 (tools only).  Prints back-to-back times and, from globaltimer stamps of
// every CTA, the median/max of each phase and the absolute chain after griddepcontrol.wait.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2605_01910_b200/csrc \
//        -Iinclude -o tools/microbench_fast tools/microbench_fast.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "score_kernels.cuh"
#include "sample_fast.cuh"

using namespace santa;
using bf16 = __nv_bfloat16;

__global__ void fill_kernel(bf16* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = __float2bfloat16(((x & 0xffff) / 65536.0f - 0.5f) * 3.4f);
  }
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 1, S = argc > 2 ? atoi(argv[2]) : 256;
  const int H = 32, Hkv = 8, D = 128, n = 32768, L = 64, NR = 4, G = 4;
  const int Cmax = n / L;
  const size_t kelems = (size_t)B * Hkv * n * D;
  std::vector<bf16*> Ks(NR), Vs(NR), qs(NR), outs(NR);
  for (int r = 0; r < NR; ++r) {
    cudaMalloc(&Ks[r], kelems * 2);
    cudaMalloc(&Vs[r], kelems * 2);
    cudaMalloc(&qs[r], (size_t)B * H * D * 2);
    cudaMalloc(&outs[r], (size_t)B * H * D * 2);
    fill_kernel<<<1024, 256>>>(Ks[r], kelems, 17 + r);
    fill_kernel<<<1024, 256>>>(Vs[r], kelems, 1017 + r);
    fill_kernel<<<8, 256>>>(qs[r], (size_t)B * H * D, 99 + r);
  }
  std::vector<int> hs(B, n);
  int* seqlens;
  cudaMalloc(&seqlens, 4 * B);
  cudaMemcpy(seqlens, hs.data(), 4 * B, cudaMemcpyHostToDevice);
  float* stash;
  float2* cstats;
  uint32_t* misc;
  unsigned long long* trace;
  cudaMalloc(&stash, (size_t)B * H * Cmax * L * 4);
  cudaMalloc(&cstats, (size_t)B * H * Cmax * 8);
  cudaMalloc(&misc, 4096);
  cudaMemset(misc, 0, 4096);
  const int ntrace = B * H * 8 * 16;
  cudaMalloc(&trace, ntrace * 8);
  unsigned long long* strace;
  cudaMalloc(&strace, 148 * 8 * 8);
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
  KvLayout kv;
  kv.page_table = nullptr;
  kv.page_size = n;
  kv.max_pages = 1;
  kv.n_kv_heads = Hkv;
  kv.page_shift = -1;
  auto sp = [&](int r, bool ho = false) {
    ScoreParams p{};
    p.q = qs[r]; p.K = Ks[r]; p.kv = kv; p.seqlens = seqlens;
    p.B = B; p.H = H; p.Hkv = Hkv;
    p.scale_log2 = 0.08838834764f * 1.4426950408889634f;
    p.stash = stash; p.cstats = cstats; p.Cmax = Cmax; p.L = L; p.stash_stride = Cmax * L;
    p.tickets = misc; p.flags = misc + 64;
    (void)ho;
    return p;
  };
  int CL = 4;
  auto pp = [&](int r, bool tr, bool ho = false) {
    SampleParams p{};
    p.stash = stash; p.cstats = cstats; p.Cmax = Cmax; p.L = L; p.stash_stride = Cmax * L;
    p.V = Vs[r]; p.kv = kv; p.seqlens = seqlens; p.B = B; p.H = H; p.Hkv = Hkv; p.S = S; p.mode = 1;
    p.seed = 0x5A17A; p.offset = r; p.out = outs[r]; p.flags = misc + 64;
    p.trace = tr ? trace : nullptr;
    p.cluster = CL;
    (void)ho;
    return p;
  };
  constexpr int NW = kStreamWarps, SPW = kStreamSlots;
  const size_t ssm = 1024 + (size_t)NW * G * L * 4 + (size_t)NW * SPW * (16384 + 16);
  auto skern = score_stream_kernel<bf16, 128, 4, NW, SPW>;
  cudaFuncSetAttribute(skern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
  auto pkern = sample_fast_kernel<bf16, 128, 4>;
  auto launch_pdl = [&](SampleParams p) {
    const size_t psm = sample_fast_smem_bytes(Cmax, D, p.cluster, S);
    cudaFuncSetAttribute(pkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(H * p.cluster, B);
    cfg.blockDim = dim3(kFastThreads);
    cfg.dynamicSmemBytes = psm;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = p.cluster;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, pkern, p) != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(cudaGetLastError()));
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](auto fn, int K) {
    for (int i = 0; i < 8; ++i) fn(i);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < K; ++i) fn(i);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / K;
  };
  printf("B=%d S=%d\nscore only      : %7.2f us\n", B, S,
         timed([&](int i) { skern<<<nsm, 32 * (NW + 1), ssm>>>(tms[i % NR], sp(i % NR)); }, 200));
  for (CL = 1; CL <= 4; CL *= 2) {
    printf("cluster %d: sample only %7.2f us", CL, timed([&](int i) { launch_pdl(pp(i % NR, false)); }, 200));
    printf("   score+sample PDL %7.2f us\n", timed([&](int i) {
             skern<<<nsm, 32 * (NW + 1), ssm>>>(tms[i % NR], sp(i % NR, true));
             launch_pdl(pp(i % NR, false, true));
           }, 200));
  }
  const char* names[11] = {"entry", "philox done", "wait done", "warp CDF blocks (bar)", "warp offsets, Z",
                           "search done (r0)", "gather done", "warp partials (bar)", "end", "-", "-"};
  for (int mode = 0; mode < 4; mode += 2) {
    CL = 4;
    const int nct = B * H * CL;
    std::vector<std::vector<double>> abs(11), dur(11);
    std::vector<double> gap, spread;
    std::vector<unsigned long long> h(ntrace);
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemset(trace, 0, ntrace * 8);
      if (mode >= 2) skern<<<nsm, 32 * (NW + 1), ssm>>>(tms[rep % NR], sp(rep % NR, true));
      launch_pdl(pp(rep % NR, true, mode >= 2));
      cudaDeviceSynchronize();
      cudaMemcpy(h.data(), trace, ntrace * 8, cudaMemcpyDeviceToHost);
      std::vector<unsigned long long> hs(148 * 8);
      cudaMemcpy(hs.data(), strace, hs.size() * 8, cudaMemcpyDeviceToHost);
      if (rep < 4) continue;
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < nct; ++c) t0 = std::min(t0, h[c * 16 + 2]);  // first wait done
      for (int c = 0; c < nct; ++c)
        for (int i = 0; i < 9; ++i) {
          if (!h[c * 16 + i]) continue;
          abs[i].push_back((double)h[c * 16 + i] - (double)t0);
          if (i) {
            int j = i - 1;
            while (j > 0 && !h[c * 16 + j]) --j;
            dur[i].push_back((double)(h[c * 16 + i] - h[c * 16 + j]));
          }
        }
    }
    printf("%s, warm=%d (CS=4): times from the first 'wait done' (ns)\n", mode >= 2 ? "score + sampler" : "sampler alone", 0);
    if (!gap.empty()) {
      std::sort(gap.begin(), gap.end());
      std::sort(spread.begin(), spread.end());
      printf("  last score warp end -> first sampler 'wait done': p50 %.0f ns; score warp end spread p50 %.0f ns\n",
             gap[gap.size() / 2], spread[spread.size() / 2]);
    }
    for (int i = 0; i < 9; ++i) {
      if (abs[i].empty()) continue;
      std::sort(abs[i].begin(), abs[i].end());
      std::sort(dur[i].begin(), dur[i].end());
      printf("  %-22s abs p50 %8.0f max %8.0f | phase p50 %7.0f max %7.0f\n", names[i], abs[i][abs[i].size() / 2],
             abs[i].back(), dur[i].empty() ? 0.0 : dur[i][dur[i].size() / 2], dur[i].empty() ? 0.0 : dur[i].back());
    }
  }
  printf("(%s)\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
