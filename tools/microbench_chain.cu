// microbench_chain.cu -- floor of the sampler's dependent chain (tools only): after a writer kernel
// has produced chunk stats and a prefix stash in L2 (as the score pass does), a 128-CTA x 256-thread
// kernel does ONLY the chain's memory round trips with trivial math in between:
//   stats (L2) -> max/sum (warp + one barrier) -> prefix block (L2) -> ballot -> V row (HBM) -> smem
//   reduction -> store.   globaltimer per phase (median over CTAs), kernel time by events.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_chain tools/microbench_chain.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void writer(float2* stats, float* stash, int nst, int nstash) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nstash; i += gridDim.x * blockDim.x) {
    stash[i] = (float)(i & 63) + 1.0f;
    if (i < nst) stats[i] = make_float2((float)((i * 7) & 15), 64.f);
  }
}

__global__ void __launch_bounds__(256, 1) chain(const float2* stats, const float* stash, const __nv_bfloat16* V,
                                               float* out, unsigned long long* tr, int nC) {
  __shared__ float sred[8];
  __shared__ double sd[8];
  __shared__ float sacc[16][128];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, head = blockIdx.x >> 2;
  unsigned long long t0 = gt();
  const float2* cs = stats + head * nC;
  float2 a = __ldcg(cs + 2 * tid), b = __ldcg(cs + 2 * tid + 1);
  float m = fmaxf(a.x, b.x);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(~0u, m, o));
  double s = (double)a.y * exp2f(a.x - m) + (double)b.y * exp2f(b.x - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if (lane == 0) { sred[warp] = m; sd[warp] = s; }
  __syncthreads();
  double Z = 0; for (int w = 0; w < 8; ++w) Z += sd[w];
  unsigned long long t1 = gt();
  // 64 samples per CTA: half-warp per sample, 4 per half-warp
  const int hw = tid >> 4, l = tid & 15;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float4 pv[4];
  int cc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    cc[u] = (int)((hw * 4 + u + blockIdx.x * 64) * 2654435761u % (unsigned)nC) + (Z < 0 ? 1 : 0);
    pv[u] = __ldcg(reinterpret_cast<const float4*>(stash + ((size_t)head * nC + cc[u]) * 64) + l);
  }
  int jj[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float t = 20.5f + u;
    const int full = __popc(__ballot_sync(~0u, pv[u].w <= t) & (0xffffu << (tid & 16)));
    jj[u] = cc[u] * 64 + min(4 * full, 63);
  }
  unsigned long long t2 = gt();
  uint4 raw[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) raw[u] = __ldg(reinterpret_cast<const uint4*>(V + ((size_t)(head >> 2) * 32768 + jj[u]) * 128) + l);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t w[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
    for (int e = 0; e < 4; ++e) { acc[2 * e] += __uint_as_float(w[e] << 16); acc[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u); }
  }
  unsigned long long t3 = gt();
  for (int e = 0; e < 8; ++e) sacc[hw][l * 8 + e] = acc[e];
  __syncthreads();
  if (tid < 128) { float r = 0; for (int i = 0; i < 16; ++i) r += sacc[i][tid]; out[blockIdx.x * 128 + tid] = r; }
  unsigned long long t4 = gt();
  if (tid == 0) { tr[blockIdx.x * 8 + 0] = t0; tr[blockIdx.x * 8 + 1] = t1; tr[blockIdx.x * 8 + 2] = t2; tr[blockIdx.x * 8 + 3] = t3; tr[blockIdx.x * 8 + 4] = t4; }
}

int main() {
  const int H = 32, nC = 512;
  float2* stats; float* stash; __nv_bfloat16* V; float* out; unsigned long long* tr;
  cudaMalloc(&stats, H * nC * 8); cudaMalloc(&stash, (size_t)H * nC * 64 * 4);
  cudaMalloc(&V, (size_t)8 * 32768 * 128 * 2 * 8); cudaMalloc(&out, 128 * 128 * 4); cudaMalloc(&tr, 128 * 8 * 8);
  char* flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<std::vector<double>> ph(4);
  float tot = 0;
  for (int rep = 0; rep < 30; ++rep) {
    cudaMemsetAsync(flush, rep, 512 << 20);  // V cold in HBM
    writer<<<148, 256>>>(stats, stash, H * nC, H * nC * 64);
    cudaEventRecord(e0);
    chain<<<128, 256>>>(stats, stash, V + (size_t)(rep % 8) * 8 * 32768 * 128, out, tr, nC);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(128 * 8);
    cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
    if (rep < 5) continue;
    tot += ms;
    for (int c = 0; c < 128; ++c) for (int i = 0; i < 4; ++i) ph[i].push_back((double)(h[c * 8 + i + 1] - h[c * 8 + i]));
  }
  const char* nm[4] = {"stats RT + max/sum + bar", "prefix block RT + ballot", "V row RT (HBM)", "smem reduce + store"};
  for (int i = 0; i < 4; ++i) { std::sort(ph[i].begin(), ph[i].end()); printf("%-28s p50 %6.0f ns  max %6.0f ns\n", nm[i], ph[i][ph[i].size() / 2], ph[i].back()); }
  printf("chain kernel (events, after writer): %.2f us  (%s)\n", tot / 25 * 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
