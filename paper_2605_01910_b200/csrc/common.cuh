// common.cuh -- small device helpers shared by the libsanta kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/santa.h"

namespace santa {

constexpr int kScoreThreads = 128; // 4 warps per score CTA
constexpr float kLog2e = 1.4426950408889634f;

// ---- Programmatic dependent launch (PDL) ---------------------------------------------
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait_primary() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// globaltimer (ns): tools-only phase traces
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- exp2 (MUFU) -----------------------------------------------------------------------
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x in fp64 for x < 1023 (chunk weights 2^(m_c - m*)), without the library exp2:
// x = n + f, n = rint(x), f in [-1/2, 1/2]; e^(f ln2) by its Taylor series to degree 13
// (truncation < 5e-18 relative) and an exact scale by 2^n.  Returns 0 below 2^-1022.
__device__ __forceinline__ double exp2_fast(double x) {
  if (!(x > -1022.0)) return 0.0;
  const double n = rint(x);
  const double g = (x - n) * 0.69314718055994530942;
  double r = 1.0 / 6227020800.0;  // 1/13!
  r = fma(r, g, 1.0 / 479001600.0);
  r = fma(r, g, 1.0 / 39916800.0);
  r = fma(r, g, 1.0 / 3628800.0);
  r = fma(r, g, 1.0 / 362880.0);
  r = fma(r, g, 1.0 / 40320.0);
  r = fma(r, g, 1.0 / 5040.0);
  r = fma(r, g, 1.0 / 720.0);
  r = fma(r, g, 1.0 / 120.0);
  r = fma(r, g, 1.0 / 24.0);
  r = fma(r, g, 1.0 / 6.0);
  r = fma(r, g, 0.5);
  r = fma(r, g, 1.0);
  r = fma(r, g, 1.0);
  return r * __longlong_as_double((long long)((int)n + 1023) << 52);
}

// ---- streaming 128-bit global loads (read once: do not allocate in L1) -----------------
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// plain weak 128-bit global load (L1-allocating)
__device__ __forceinline__ uint4 ldg_plain(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ float4 ldcg_f4(const void* p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// ---- element conversion ------------------------------------------------------------------
template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
  static __device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
  static __device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
  static __device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};
template <> struct Elem<__half> {
  static __device__ __forceinline__ float lo(uint32_t w) {
    return __half2float(__ushort_as_half((unsigned short)(w & 0xffffu)));
  }
  static __device__ __forceinline__ float hi(uint32_t w) {
    return __half2float(__ushort_as_half((unsigned short)(w >> 16)));
  }
  static __device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
  static __device__ __forceinline__ __half from_f(float x) { return __float2half_rn(x); }
};
template <> struct Elem<float> {
  static __device__ __forceinline__ float to_f(float x) { return x; }
  static __device__ __forceinline__ float from_f(float x) { return x; }
};

// ---- legacy warp-level tensor-core MMA: D[16x8] += A[16x16] * B[16x8], fp32 accumulate --
template <typename T> struct Mma;
template <> struct Mma<__nv_bfloat16> {
  static __device__ __forceinline__ void run(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
};
template <> struct Mma<__half> {
  static __device__ __forceinline__ void run(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
};

// ---- KV addressing (head-major, optionally paged) ------------------------------------------
struct KvLayout {
  const int32_t* page_table;  // NULL => contiguous [B, Hkv, page_size(=max_seqlen), D]
  int32_t page_size;
  int32_t max_pages;
  int32_t n_kv_heads;
  int32_t page_shift;         // log2(page_size) if a power of two, else -1 (paged only)
  // element offset of row `t` (token) of (b, kvh); the row is D contiguous elements
  __device__ __forceinline__ int64_t row(int b, int kvh, int t, int D) const {
    if (!page_table) return (((int64_t)b * n_kv_heads + kvh) * page_size + t) * D;
    int page, within;
    if (page_shift >= 0) {
      page = t >> page_shift;
      within = t & (page_size - 1);
    } else {
      page = t / page_size;
      within = t - page * page_size;
    }
    const int64_t phys = (int64_t)__ldg(page_table + (int64_t)b * max_pages + page);
    return ((phys * n_kv_heads + kvh) * (int64_t)page_size + within) * D;
  }
};

// ---- warp scans ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_incl_scan(float v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ double warp_incl_scan_d(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

}  // namespace santa
