// microbench_fp64.cu -- dependent-chain latency (cycles) of a few ops the sampler uses (tools only).
#include <cstdio>
__global__ void k(float* fo, double* dout, long long* cyc, float x, double y) {
  long long t0, t1;
  double d = y;
  float f = x;
  // DADD chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) d = d + 1e-9;
  t1 = clock64();
  cyc[0] = (t1 - t0);
  // F2F.F64.F32 + F2F.F32.F64 chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) f = (float)((double)f * 1.0000001);
  t1 = clock64();
  cyc[1] = (t1 - t0);
  // DMUL chain
  double m = y;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) m = m * 1.0000000001;
  t1 = clock64();
  cyc[2] = (t1 - t0);
  // FFMA chain (reference)
  float g = x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) g = g * 1.0000001f + 1e-9f;
  t1 = clock64();
  cyc[3] = (t1 - t0);
  // MUFU.EX2 chain
  float e = x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e)); e = r * 1e-3f; }
  t1 = clock64();
  cyc[4] = (t1 - t0);
  // DDIV chain
  double q = y;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) q = 1.0 / (q + 1.5);
  t1 = clock64();
  cyc[5] = (t1 - t0) * 4;
  fo[0] = f + g + e;
  dout[0] = d + m + q;
}
int main() {
  float* fo; double* dd; long long* c;
  cudaMalloc(&fo, 4); cudaMalloc(&dd, 8); cudaMalloc(&c, 64);
  k<<<1, 32>>>(fo, dd, c, 0.5f, 0.25);
  k<<<1, 32>>>(fo, dd, c, 0.5f, 0.25);
  long long h[6];
  cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  const char* n[6] = {"DADD", "F2F f32->f64->f32 + DMUL", "DMUL", "FFMA", "MUFU.EX2 + FMUL", "DDIV (per 1/4 iter)"};
  for (int i = 0; i < 6; ++i) printf("%-28s %6.1f cycles per dependent op\n", n[i], h[i] / 256.0);
  return 0;
}
