// microbench_lat.cu -- dependent-chain latencies of the instructions the sampler chain is made of
// (tools only): DFMA, DADD, FFMA, SHFL (32/64-bit), LDS.64, L2-hit LDG, __syncthreads (256 threads),
// globaltimer read, DDIV, MUFU.EX2.  clock64 cycles per operation.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_lat tools/microbench_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void lat(double* dout, float* fout, long long* res, const double* gbuf, int n) {
  __shared__ double sm[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  double x = dout[0], y = 1.0000001;
  float fx = fout[0], fy = 1.0000001f;
  long long t0, t1;
  const int N = 256;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (tid == 0) res[0] = (t1 - t0) / N;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x + y;
  t1 = clock64();
  if (tid == 0) res[1] = (t1 - t0) / N;
  // FFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) fx = fmaf(fx, fy, 1e-9f);
  t1 = clock64();
  if (tid == 0) res[2] = (t1 - t0) / N;
  // SHFL 32 chain
  int v = tid;
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
  t1 = clock64();
  if (tid == 0) res[3] = (t1 - t0) / N;
  // SHFL 64 (double) chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  t1 = clock64();
  if (tid == 0) res[4] = (t1 - t0) / N;
  // LDS.64 pointer chase
  int idx = tid & 1023;
  t0 = clock64();
  for (int i = 0; i < N; ++i) idx = (int)sm[idx];
  t1 = clock64();
  if (tid == 0) res[5] = (t1 - t0) / N;
  // L2-hit LDG chase (buffer small, .cg)
  int gi = tid % n;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) gi = (int)__ldcg(gbuf + gi);
  t1 = clock64();
  if (tid == 0) res[6] = (t1 - t0) / 64;
  // __syncthreads
  t0 = clock64();
  for (int i = 0; i < 64; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) res[7] = (t1 - t0) / 64;
  // globaltimer read
  unsigned long long g = 0;
  t0 = clock64();
  for (int i = 0; i < 64; ++i) g += gt();
  t1 = clock64();
  if (tid == 0) res[8] = (t1 - t0) / 64;
  // DDIV chain
  t0 = clock64();
  for (int i = 0; i < 64; ++i) x = y / x;
  t1 = clock64();
  if (tid == 0) res[9] = (t1 - t0) / 64;
  // ex2.approx chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    float r;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fx));
    fx = r * 0.5f;
  }
  t1 = clock64();
  if (tid == 0) res[10] = (t1 - t0) / N;
  // cvt f32->f64 + DMUL chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { x = (double)fx * x; fx = (float)x; }
  t1 = clock64();
  if (tid == 0) res[11] = (t1 - t0) / N;
  dout[tid] = x + (double)g + idx + gi + v;
  fout[tid] = fx;
}

int main() {
  double* d; float* f; long long* r; double* g;
  cudaMalloc(&d, 8 * 1024); cudaMalloc(&f, 4 * 1024); cudaMalloc(&r, 8 * 16); cudaMalloc(&g, 8 * 4096);
  double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (double)((i * 1031 + 7) % 4096);
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemset(d, 0, 8 * 1024); cudaMemset(f, 0, 4 * 1024);
  for (int nt : {32, 256}) {
    lat<<<1, nt>>>(d, f, r, g, 4096);
    lat<<<1, nt>>>(d, f, r, g, 4096);
    long long hr[16];
    cudaMemcpy(hr, r, sizeof(hr), cudaMemcpyDeviceToHost);
    const char* nm[12] = {"DFMA", "DADD", "FFMA", "SHFL32", "SHFL64+DADD", "LDS.64 chase", "LDG L2 chase", "__syncthreads",
                          "globaltimer", "DDIV", "EX2+FMUL", "F2F.F64+DMUL+F2F"};
    printf("threads %d:\n", nt);
    for (int i = 0; i < 12; ++i) printf("  %-18s %lld cycles\n", nm[i], hr[i]);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz (%s)\n", clk, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
