// microbench_sample.cu -- phase timing of the sample/gather kernel (tools only).
// Config-2 shape (B=1, H=32, H_kv=8, d=128, bf16, n=32768, S=256 stratified, L=64).  Runs the
// streaming score kernel, then the sampler with its globaltimer trace enabled, and prints the
// median duration of each phase over CTAs and repetitions, plus back-to-back timings.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2605_01910_b200/csrc \
//        -o tools/microbench_sample tools/microbench_sample.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fused_kernel_gridsync.cuh"

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
  const int B = 1, H = 32, Hkv = 8, D = 128, n = 32768, L = 64, S = 256, NR = 4, G = 4;
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
  int* seqlens;
  cudaMalloc(&seqlens, 4);
  cudaMemcpy(seqlens, &n, 4, cudaMemcpyHostToDevice);
  float* stash;
  float2* cstats;
  uint32_t* misc;
  unsigned long long* trace;
  cudaMalloc(&stash, (size_t)B * H * Cmax * L * 4);
  cudaMalloc(&cstats, (size_t)B * H * Cmax * 8);
  cudaMalloc(&misc, 4096);
  const int ntrace = B * H * 16 + 148 * 8;
  cudaMalloc(&trace, ntrace * 8);
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
  auto sp = [&](int r) {
    ScoreParams p{};
    p.q = qs[r]; p.K = Ks[r]; p.kv = kv; p.seqlens = seqlens;
    p.B = B; p.H = H; p.Hkv = Hkv;
    p.scale_log2 = 0.08838834764f * 1.4426950408889634f;
    p.stash = stash; p.cstats = cstats; p.Cmax = Cmax; p.L = L; p.stash_stride = Cmax * L;
    p.tickets = misc; p.flags = misc + 64;
    return p;
  };
  int CL = 1;
  auto pp = [&](int r, bool tr) {
    SampleParams p{};
    p.stash = stash; p.cstats = cstats; p.Cmax = Cmax; p.L = L; p.stash_stride = Cmax * L;
    p.V = Vs[r]; p.kv = kv; p.seqlens = seqlens; p.B = B; p.H = H; p.Hkv = Hkv; p.S = S; p.mode = 1;
    p.seed = 0x5A17A; p.offset = r; p.out = outs[r]; p.flags = misc + 64;
    p.trace = tr ? trace : nullptr;
    p.cluster = CL;
    return p;
  };
  constexpr int NW = kStreamWarps, SPW = kStreamSlots;
  const size_t ssm = 1024 + (size_t)NW * G * L * 4 + (size_t)NW * SPW * (16384 + 16);
  auto skern = score_stream_kernel<bf16, 128, 4, NW, SPW>;
  cudaFuncSetAttribute(skern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
  const size_t psm = getenv("PAD") ? (size_t)120 * 1024 : (size_t)Cmax * 16 + (size_t)S * 16 + 17 * 128 * 4 + 64;
  auto pkern = sample_gather_kernel<bf16, 128, 4>;
  cudaFuncSetAttribute(pkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
  auto launch_pdl = [&](SampleParams p) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(H * p.cluster, B);
    cfg.blockDim = dim3(kSampleThreads);
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
    cudaLaunchKernelEx(&cfg, pkern, p);
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](auto fn, int K) {
    for (int i = 0; i < 4; ++i) fn(i);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < K; ++i) fn(i);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / K;
  };
  printf("score only      : %7.2f us\n", timed([&](int i) { skern<<<nsm, 32 * (NW + 1), ssm>>>(tms[i % NR], sp(i % NR)); }, 40));
  for (CL = 1; CL <= 8; CL *= 2) {
    printf("cluster %d: sample only %7.2f us", CL, timed([&](int i) { launch_pdl(pp(i % NR, false)); }, 40));
    printf("   score+sample PDL %7.2f us\n", timed([&](int i) {
             skern<<<nsm, 32 * (NW + 1), ssm>>>(tms[i % NR], sp(i % NR));
             launch_pdl(pp(i % NR, false));
           }, 40));
  }
  CL = 1;
  // fused kernel: one cooperative launch
  {
    constexpr int NT = 32 * (NW + 1);
    const size_t fsm = ssm;
    auto fk = santa_fused_kernel<bf16, 128, 4, NW, SPW>;
    cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
    auto launch_fused = [&](int r, int cl, bool tr) {
      SampleParams p = pp(r, tr);
      p.cluster = cl;
      unsigned long long* sp_part;
      static float* split = nullptr;
      if (!split) cudaMalloc(&split, (size_t)B * H * 8 * 128 * 4);
      p.split_partial = split;
      (void)sp_part;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nsm);
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = fsm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, fk, tms[r], sp(r), p);
    };
    for (int cl = 1; cl <= 8; cl *= 2)
      printf("fused (CS=%d)    : %7.2f us\n", cl, timed([&](int i) { launch_fused(i % NR, cl, false); }, 40));
    std::vector<unsigned long long> h(ntrace);
    std::vector<std::vector<double>> ph(5);
    for (int rep = 0; rep < 12; ++rep) {
      launch_fused(rep % NR, 4, true);
      cudaDeviceSynchronize();
      cudaMemcpy(h.data(), trace, ntrace * 8, cudaMemcpyDeviceToHost);
      if (rep < 2) continue;
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < nsm; ++c) t0 = std::min(t0, h[B * H * 16 + c * 8 + 0]);
      for (int c = 0; c < nsm; ++c)
        for (int i = 0; i < 5; ++i) ph[i].push_back((double)(h[B * H * 16 + c * 8 + i + 1] - t0));
    }
    {
      std::vector<std::vector<double>> q(6);
      for (int rep = 0; rep < 10; ++rep) {
        launch_fused(rep % NR, 4, true);
        cudaDeviceSynchronize();
        cudaMemcpy(h.data(), trace, ntrace * 8, cudaMemcpyDeviceToHost);
        for (int c = 0; c < B * H; ++c)
          for (int i = 0; i < 6; ++i) q[i].push_back((double)(h[c * 16 + i + 1] - h[c * 16 + i]));
      }
      const char* pn[6] = {"thresholds", "pdl wait", "cstats+max", "CDF", "chunk search", "search+gather"};
      for (int i = 0; i < 6; ++i) {
        std::sort(q[i].begin(), q[i].end());
        printf("fused item phase %-14s median %7.0f ns\n", pn[i], q[i][q[i].size() / 2]);
      }
    }
    const char* nm[5] = {"score done", "grid.sync #1", "sample item done", "grid.sync #2", "end"};
    for (int i = 0; i < 5; ++i) {
      std::sort(ph[i].begin(), ph[i].end());
      printf("fused t(%-16s) median %8.0f ns  max %8.0f ns (from first CTA start)\n", nm[i], ph[i][ph[i].size() / 2],
             ph[i].back());
    }
  }
  // phase trace in three settings
  const char* names[7] = {"thresholds (Philox)", "griddepcontrol.wait", "cstats load + max", "fp64 CDF scan+clamp",
                          "chunk search (smem)", "in-chunk search+gather", "reduce + store"};
  for (int mode = 0; mode < 3; ++mode) {
    std::vector<std::vector<double>> ph(7);
    std::vector<unsigned long long> h(ntrace);
    for (int rep = 0; rep < 20; ++rep) {
      if (mode != 2) skern<<<nsm, 32 * (NW + 1), ssm>>>(tms[rep % NR], sp(rep % NR));
      if (mode == 1) cudaDeviceSynchronize();
      launch_pdl(pp(rep % NR, true));
      cudaDeviceSynchronize();
      cudaMemcpy(h.data(), trace, ntrace * 8, cudaMemcpyDeviceToHost);
      if (rep < 4) continue;
      for (int c = 0; c < B * H; ++c)
        for (int i = 0; i < 7; ++i) ph[i].push_back((double)(h[c * 16 + i + 1] - h[c * 16 + i]));
    }
    printf("---- %s ----\n", mode == 0 ? "score -> sample (PDL)" : mode == 1 ? "score; sync; sample" : "sample only (stash hot)");
    {
      std::vector<double> a, b2, c2;
      for (int c = 0; c < B * H; ++c) {
        if (!h[c * 16 + 8] || !h[c * 16 + 9]) continue;
        a.push_back((double)(h[c * 16 + 8] - h[c * 16 + 5]));
        b2.push_back((double)(h[c * 16 + 9] - h[c * 16 + 8]));
        c2.push_back((double)(h[c * 16 + 6] - h[c * 16 + 9]));
      }
      std::sort(a.begin(), a.end()); std::sort(b2.begin(), b2.end()); std::sort(c2.begin(), c2.end());
      if (!a.empty())
        printf("  (last rep) stash+ballots %6.0f ns | V gather+add %6.0f ns | reduce barrier %6.0f ns (medians)\n",
               a[a.size() / 2], b2[b2.size() / 2], c2[c2.size() / 2]);
    }
    for (int i = 0; i < 7; ++i) {
      std::sort(ph[i].begin(), ph[i].end());
      printf("phase %-22s median %8.0f ns   p90 %8.0f ns\n", names[i], ph[i][ph[i].size() / 2],
             ph[i][ph[i].size() * 9 / 10]);
    }
  }
  printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
