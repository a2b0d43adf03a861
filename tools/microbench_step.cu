// microbench_step.cu -- timeline of the single-launch step kernel (tools only, not part of
// libsanta).  Config-2 shape (B=1, H=32, H_kv=8, d=128, bf16, n=32768, S=256 stratified, L=64)
// by default; `./microbench_step B` runs batch B.  Prints back-to-back launch times and, for one
// traced launch inside a back-to-back run, the per-CTA / per-unit / per-item %globaltimer phases.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2605_01910_b200/csrc \
//        -o tools/microbench_step tools/microbench_step.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "step_kernel.cuh"

using namespace santa;
using bf16 = __nv_bfloat16;

__global__ void fill_kernel(bf16* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = __float2bfloat16(((x & 0xffff) / 65536.0f - 0.5f) * 3.4f);
  }
}

static void stat(const char* name, std::vector<double> v) {
  if (v.empty()) return;
  std::sort(v.begin(), v.end());
  printf("  %-34s n=%4zu  min %8.2f  p50 %8.2f  p90 %8.2f  max %8.2f us\n", name, v.size(), v.front(),
         v[v.size() / 2], v[(v.size() * 9) / 10], v.back());
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 1;
  const int H = 32, Hkv = 8, D = 128, n = 32768, L = 64, S = 256, NR = B == 1 ? 4 : 1, G = 4;
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
  std::vector<int> sl(B, n);
  int* seqlens;
  cudaMalloc(&seqlens, 4 * B);
  cudaMemcpy(seqlens, sl.data(), 4 * B, cudaMemcpyHostToDevice);
  float* stash;
  float2* cstats;
  uint32_t *misc, *sync, *sstash;
  ulonglong2* rec;
  unsigned long long* part;
  cudaMalloc(&stash, (size_t)B * H * Cmax * L * 4);
  cudaMalloc(&cstats, (size_t)B * H * Cmax * 8);
  cudaMalloc(&misc, 4096);
  const size_t nsync = 2 + B * H;
  cudaMalloc(&sync, nsync * 4);
  cudaMemset(sync, 0, nsync * 4);
  cudaMalloc(&rec, (size_t)B * H * Cmax * 16);
  cudaMemset(rec, 0, (size_t)B * H * Cmax * 16);
  cudaMalloc(&sstash, (size_t)B * H * Cmax * 64 * 4);
  cudaMemset(sstash, 0, (size_t)B * H * Cmax * 64 * 4);
  cudaMalloc(&part, (size_t)B * H * 16 * D * 8);
  cudaMemset(part, 0, (size_t)B * H * 16 * D * 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* trace;
  const size_t ntrace = (size_t)nsm * kTraceStride + B * Hkv;
  cudaMalloc(&trace, ntrace * 8);
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
  int CS = 1;
  while (CS * 2 <= 16 && B * H * CS * 2 <= 148 && CS * 2 * 32 <= S) CS *= 2;
  auto sp = [&](int r) {
    ScoreParams p{};
    p.q = qs[r]; p.K = Ks[r]; p.kv = kv; p.seqlens = seqlens;
    p.B = B; p.H = H; p.Hkv = Hkv;
    p.scale_log2 = 0.08838834764f * 1.4426950408889634f;
    p.stash = stash; p.cstats = cstats; p.Cmax = Cmax; p.L = L; p.stash_stride = Cmax * L;
    p.tickets = misc; p.flags = misc + 64;
    return p;
  };
  auto pp = [&](int r) {
    SampleParams p{};
    p.stash = stash; p.cstats = cstats; p.Cmax = Cmax; p.L = L; p.stash_stride = Cmax * L;
    p.V = Vs[r]; p.kv = kv; p.seqlens = seqlens; p.B = B; p.H = H; p.Hkv = Hkv; p.S = S; p.mode = 1;
    p.seed = 0x5A17A; p.offset = r; p.out = outs[r]; p.flags = misc + 64;
    p.cluster = CS;
    return p;
  };
  auto sy = [&](bool tr) {
    StepSync s;
    s.epoch = sync;
    s.exit_ticket = sync + 1;
    s.head_ticket = sync + 2;
    s.rec = rec;
    s.stash = sstash;
    s.part = part;
    s.trace = tr ? trace : nullptr;
    return s;
  };
  constexpr int NW = kStepConsumers, NSW = kStepSamplers, NT = 32 * (NW + 1 + NSW), SPW = kStepSlots;
  struct Var { const char* name; int var; int coop; };
  const Var vars[] = {{"stream only (coop)", 3, 1}, {"stream only (non-coop)", 3, 0}, {"score, no samplers", 2, 1},
                      {"full", 0, 1}};
  auto get = [&](int var) -> void (*)(CUtensorMap, ScoreParams, SampleParams, StepSync) {
    if (var == 0) return santa_step_kernel<bf16, 128, 4, NW, SPW, NSW, 0>;
    if (var == 2) return santa_step_kernel<bf16, 128, 4, NW, SPW, NSW, 2>;
    return santa_step_kernel<bf16, 128, 4, NW, SPW, NSW, 3>;
  };
  Var cur = vars[3];
  const size_t smem = step_score_smem_bytes(D, G, NW, SPW) + step_sample_smem_bytes(Cmax, (S + CS - 1) / CS, D);
  auto launch = [&](int r, bool tr) {
    auto kern = get(cur.var);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = cur.coop;
    return cudaLaunchKernelEx(&cfg, kern, tms[r], sp(r), pp(r), sy(tr));
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
  printf("B=%d n=%d S=%d CS=%d smem=%zu (%s)\n", B, n, S, CS, smem, cudaGetErrorString(launch(0, false)));
  cudaDeviceSynchronize();
  {
    uint32_t ep[2], fl;
    unsigned long long r[4];
    uint32_t q[4];
    cudaMemcpy(ep, sync, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&fl, misc + 64, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(r, rec + 511, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(r + 2, rec + 0, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(q, sstash + 511 * 64 + 60, 16, cudaMemcpyDeviceToHost);
    printf("debug: epoch %u exit %u flags %x rec[511] tags %x %x rec[0] tags %x %x stash tags %x %x\n", ep[0], ep[1],
           fl, (unsigned)(r[0] >> 32), (unsigned)(r[1] >> 32), (unsigned)(r[2] >> 32), (unsigned)(r[3] >> 32),
           q[0] >> 24, q[3] >> 24);
  }
  if (argc > 3) {  // profiling mode: the full kernel only
    cur = vars[3];
    for (int i = 0; i < 8; ++i) launch(i % NR, false);
    cudaDeviceSynchronize();
    printf("profile mode done (%s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  for (const Var& v : vars) {
    cur = v;
    const double us = timed([&](int i) { launch(i % NR, false); }, 40);
    printf("step kernel back-to-back [%-24s]: %8.2f us/launch\n", v.name, us);
  }
  const int tv = argc > 2 ? atoi(argv[2]) : 3;
  cur = vars[tv];
  printf("trace variant: %s\n", cur.name);
  cudaMemset(trace, 0, ntrace * 8);
  for (int i = 0; i < 6; ++i) launch(i % NR, i == 4);
  cudaDeviceSynchronize();
  printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
  std::vector<unsigned long long> tr(ntrace);
  cudaMemcpy(tr.data(), trace, ntrace * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < nsm; ++c) t0 = std::min(t0, tr[(size_t)c * kTraceStride]);
  auto rel = [&](unsigned long long t) { return t ? (double)(t - t0) * 1e-3 : -1.0; };
  std::vector<double> start, prod, first, last;
  for (int c = 0; c < nsm; ++c) {
    const unsigned long long* x = &tr[(size_t)c * kTraceStride];
    start.push_back(rel(x[0]));
    prod.push_back(rel(x[1]));
    double f = 1e30, l = 0;
    for (int j = 0; j < NW; ++j) {
      if (x[14 + j]) f = std::min(f, rel(x[14 + j]));
      l = std::max(l, rel(x[2 + j]));
    }
    first.push_back(f);
    last.push_back(l);
  }
  printf("timeline of one launch (t=0: first CTA start):\n");
  stat("CTA start", start);
  stat("first stage landed (per CTA)", first);
  stat("producer done issuing", prod);
  stat("consumers done (per CTA)", last);
  std::vector<double> tw, tmm, tep, nch;
  for (int c = 0; c < nsm; ++c)
    for (int j = 0; j < NW; ++j) {
      const unsigned long long* x = &tr[(size_t)c * kTraceStride];
      tw.push_back(x[64 + 3 * j] * 1e-3);
      tmm.push_back(x[65 + 3 * j] * 1e-3);
      tep.push_back(x[66 + 3 * j] * 1e-3);
      nch.push_back((double)x[88 + j]);
    }
  stat("consumer warp: waiting for stages", tw);
  stat("consumer warp: LDS + MMA", tmm);
  stat("consumer warp: epilogue + publish", tep);
  stat("consumer warp: chunks (count)", nch);
  const char* pn[10] = {"wait start", "wait done", "stats loaded", "CDF done", "chunk search done",
                        "stash validated", "indices (ballots)", "gather done", "out/partial written", "item end"};
  const int order[10] = {0, 1, 2, 3, 4, 8, 9, 5, 6, 7};
  std::vector<double> abs_[10], dur[10];
  for (int c = 0; c < nsm; ++c)
    for (int i = 0; i < 3; ++i) {
      const unsigned long long* x = &tr[(size_t)c * kTraceStride + 24 + 10 * i];
      if (!x[0] || !x[7]) continue;
      for (int k = 0; k < 10; ++k) {
        abs_[k].push_back(rel(x[order[k]]));
        if (k) dur[k].push_back((double)(x[order[k]] - x[order[k - 1]]) * 1e-3);
      }
    }
  {
    std::vector<double> a1, a2, a3;
    for (int c = 0; c < nsm; ++c)
      for (int i = 0; i < 3; ++i) {
        const unsigned long long* x = &tr[(size_t)c * kTraceStride + 24 + 10 * i];
        const unsigned long long* y = &tr[(size_t)c * kTraceStride + 120 + 2 * i];
        if (!x[0] || !x[7] || !y[0]) continue;
        a1.push_back((double)(y[0] - x[2]) * 1e-3);
        a2.push_back((double)(y[1] - y[0]) * 1e-3);
        a3.push_back((double)(x[3] - y[1]) * 1e-3);
      }
    stat("CDF: weights (ex2, fp64 mul)", a1);
    stat("CDF: warp scans + group bar", a2);
    stat("CDF: offsets, 1/Z, F, bar", a3);
  }
  printf("sampler items, absolute times:\n");
  for (int k = 0; k < 10; ++k) stat(pn[k], abs_[k]);
  {  // the three items that finish last: their own timelines
    std::vector<std::pair<unsigned long long, std::pair<int, int>>> ends;
    for (int c = 0; c < nsm; ++c)
      for (int i = 0; i < 3; ++i) {
        const unsigned long long* x = &tr[(size_t)c * kTraceStride + 24 + 10 * i];
        if (x[0] && x[7]) ends.push_back({x[7], {c, i}});
      }
    std::sort(ends.begin(), ends.end());
    for (size_t e = ends.size() >= 3 ? ends.size() - 3 : 0; e < ends.size(); ++e) {
      const int c = ends[e].second.first, i = ends[e].second.second;
      const unsigned long long* x = &tr[(size_t)c * kTraceStride + 24 + 10 * i];
      const unsigned long long* y = &tr[(size_t)c * kTraceStride + 120 + 2 * i];
      printf("  last item (CTA %d):", c);
      for (int k = 0; k < 10; ++k) printf(" %s=%.2f", pn[k], rel(x[order[k]]));
      printf(" | cdf: weights=%.2f scans=%.2f\n", rel(y[0]), rel(y[1]));
    }
  }
  printf("sampler items, phase durations (from the previous point):\n");
  for (int k = 1; k < 10; ++k) stat(pn[k], dur[k]);
  return 0;
}
