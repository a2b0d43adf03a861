// peer_exchange.cu -- one-shot peer-memory collectives for the sequence-sharded step (config 4,
// SURVEY 8(e) / NEXT-3): the all-gather of the per-shard statistics (m_r, L_r) and the SUM of the
// per-shard partial outputs, as ONE kernel each that stores straight into every peer's exchange
// buffer over NVLink (P2P stores through CUDA-IPC mappings) and then waits on per-(source, block)
// flags -- no NCCL launch, no proxy thread, one kernel boundary per exchange.  The reduction is
// summed in fixed rank order from the gathered slots, so every rank gets the same bits (NCCL's
// ring / tree order is not fixed across world sizes).  See include/santa.h, "Peer-memory exchange".
//
// Buffer layout (identical on every rank; the caller zeroes it once):
//   [0, 256)        error word (bit SANTA_FLAG_PEER_TIMEOUT) + padding
//   [256, 4352)     flags u32 [2 parities][8 sources][64 blocks]
//   [8192, ...)     data [2 parities][world slots][slot_bytes]
// Call e (epoch, >= 1, +1 per call on the group) uses parity e & 1.  A rank writes parity p of
// call e into a peer only after its own call e-1 finished (stream order), and call e-1 finished only
// after every peer pushed call e-1, which each peer did after consuming call e-2 (parity p) -- so
// two parities are enough and no slot is overwritten while it is read.
#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "santa.h"

namespace {

constexpr int kMaxWorld = 8;
constexpr int kMaxBlk = 64;
constexpr size_t kFlagOff = 256;
constexpr size_t kDataOff = 8192;
constexpr int kThreads = 256;
constexpr size_t kMinBlkBytes = 2048;      // payload bytes per CTA before another CTA is worth it
constexpr unsigned long long kTimeoutNs = 2000000000ull;  // give up a wait after 2 s (error word)

struct PeerArgs {
  char* bufs[kMaxWorld];          // every rank's exchange buffer as addressable from this process
  const char* src[kMaxWorld];     // per emulated local rank: payload (device)
  char* dst[kMaxWorld];           // per emulated local rank: result (device)
  int rank[kMaxWorld];            // per emulated local rank: its rank id
  int world;
  int nblk;                       // CTAs per local rank; CTA k owns payload bytes [k*chunk, ...)
  size_t bytes;                   // payload bytes per rank (multiple of 16)
  size_t chunk;                   // bytes per CTA (multiple of 16)
  size_t slot;                    // slot bytes in the data region
  uint32_t epoch;
  int op;                         // 0: all-gather (dst [world][bytes]); 1: fp32 SUM (dst [bytes])
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t* flag_ptr(char* buf, int parity, int src, int blk) {
  return reinterpret_cast<uint32_t*>(buf + kFlagOff) + ((size_t)parity * kMaxWorld + src) * kMaxBlk + blk;
}
__device__ __forceinline__ char* slot_ptr(char* buf, const PeerArgs& a, int parity, int src) {
  return buf + kDataOff + ((size_t)parity * a.world + src) * a.slot;
}

// grid (nblk, n_local): CTA (k, l) acts for local rank l on payload block k.
// 1. push: store the block into slot[rank] of EVERY rank's buffer (own included), then one thread
//    per destination releases flag[parity][rank][k] = epoch there (bar.sync orders the CTA's stores
//    before the release; release.sys makes them visible to the peer GPU before the flag);
// 2. wait: one thread per source acquires flag[parity][src][k] == epoch in the OWN buffer;
// 3. consume block k from the own buffer's slots (L2 loads: the slots were written by other GPUs).
__global__ void __launch_bounds__(kThreads) peer_exchange_kernel(const PeerArgs a) {
  const int k = blockIdx.x, l = blockIdx.y;
  const int rank = a.rank[l];
  const int parity = (int)(a.epoch & 1u);
  const size_t lo = (size_t)k * a.chunk;
  const size_t hi = lo + a.chunk < a.bytes ? lo + a.chunk : a.bytes;
  const size_t n16 = hi > lo ? (hi - lo) / 16 : 0;
  const uint4* s = reinterpret_cast<const uint4*>(a.src[l] + lo);
  for (int j = 0; j < a.world; ++j) {
    const int dstr = (rank + 1 + j) % a.world;          // own slot last; peers in rotated order
    uint4* d = reinterpret_cast<uint4*>(slot_ptr(a.bufs[dstr], a, parity, rank) + lo);
    for (size_t i = threadIdx.x; i < n16; i += kThreads) d[i] = __ldg(s + i);
  }
  __syncthreads();
  if (threadIdx.x < a.world) st_release_sys(flag_ptr(a.bufs[threadIdx.x], parity, rank, k), a.epoch);
  char* own = a.bufs[rank];
  __shared__ int timed_out;
  if (threadIdx.x == 0) timed_out = 0;
  __syncthreads();
  if (threadIdx.x < a.world) {
    const uint32_t* f = flag_ptr(own, parity, threadIdx.x, k);
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(f) != a.epoch) {
      if (globaltimer() - t0 > kTimeoutNs) {
        timed_out = 1;
        atomicOr(reinterpret_cast<unsigned int*>(own), (unsigned int)SANTA_FLAG_PEER_TIMEOUT);
        break;
      }
    }
  }
  __syncthreads();
  if (timed_out) return;
  if (a.op == 0) {
    for (int r = 0; r < a.world; ++r) {
      const uint4* sl = reinterpret_cast<const uint4*>(slot_ptr(own, a, parity, r) + lo);
      uint4* d = reinterpret_cast<uint4*>(a.dst[l] + (size_t)r * a.bytes + lo);
      for (size_t i = threadIdx.x; i < n16; i += kThreads) d[i] = __ldcg(sl + i);
    }
  } else {
    float4* d = reinterpret_cast<float4*>(a.dst[l] + lo);
    for (size_t i = threadIdx.x; i < n16; i += kThreads) {
      float4 acc = __ldcg(reinterpret_cast<const float4*>(slot_ptr(own, a, parity, 0) + lo) + i);
      for (int r = 1; r < a.world; ++r) {         // fixed rank order: identical bits on every rank
        const float4 v = __ldcg(reinterpret_cast<const float4*>(slot_ptr(own, a, parity, r) + lo) + i);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      d[i] = acc;
    }
  }
}

struct Nvtx {
  explicit Nvtx(const char* n) { nvtxRangePushA(n); }
  ~Nvtx() { nvtxRangePop(); }
};

size_t slot_bytes(int world, size_t buf_bytes) {
  if (world < 1 || world > kMaxWorld || buf_bytes <= kDataOff) return 0;
  return ((buf_bytes - kDataOff) / (2 * (size_t)world)) / 256 * 256;
}

santa_status run(const santa_peer_group* g, int32_t n_local, const int32_t* ranks, const void* const* src,
                 void* const* dst, size_t bytes, uint32_t epoch, int op, void* stream) {
  if (!g || !ranks || !src || !dst) return SANTA_ERR_INVALID_ARG;
  if (g->world < 1 || g->world > kMaxWorld || n_local < 1 || n_local > g->world) return SANTA_ERR_INVALID_ARG;
  if (epoch == 0 || bytes == 0) return SANTA_ERR_INVALID_ARG;
  if (bytes % 16) return SANTA_ERR_ALIGNMENT;
  const size_t slot = slot_bytes(g->world, g->buf_bytes);
  if (bytes > slot) return SANTA_ERR_WORKSPACE;
  PeerArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int r = 0; r < g->world; ++r) {
    if (!g->bufs[r] || (reinterpret_cast<uintptr_t>(g->bufs[r]) & 255)) return SANTA_ERR_ALIGNMENT;
    a.bufs[r] = static_cast<char*>(g->bufs[r]);
  }
  uint32_t seen = 0;
  for (int l = 0; l < n_local; ++l) {
    if (ranks[l] < 0 || ranks[l] >= g->world || (seen >> ranks[l]) & 1u) return SANTA_ERR_INVALID_ARG;
    seen |= 1u << ranks[l];
    if (!src[l] || !dst[l]) return SANTA_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(src[l]) | reinterpret_cast<uintptr_t>(dst[l])) & 15) return SANTA_ERR_ALIGNMENT;
    a.rank[l] = ranks[l];
    a.src[l] = static_cast<const char*>(src[l]);
    a.dst[l] = static_cast<char*>(dst[l]);
  }
  size_t nblk = (bytes + kMinBlkBytes - 1) / kMinBlkBytes;
  if (nblk > (size_t)kMaxBlk) nblk = kMaxBlk;
  size_t chunk = ((bytes + nblk - 1) / nblk + 15) / 16 * 16;
  nblk = (bytes + chunk - 1) / chunk;
  a.world = g->world;
  a.nblk = (int)nblk;
  a.bytes = bytes;
  a.chunk = chunk;
  a.slot = slot;
  a.epoch = epoch;
  a.op = op;
  // cooperative when n_local > 1 (all ranks of a group emulated in one launch on one GPU): the CTAs
  // wait on one another, so they must be co-resident -- which a cooperative launch guarantees (or
  // refuses); with n_local == 1 they only wait on other GPUs and a plain launch is cheaper.
  void* args[] = {&a};
  const dim3 grid((unsigned)nblk, (unsigned)n_local);
  const cudaError_t e =
      n_local > 1 ? cudaLaunchCooperativeKernel(reinterpret_cast<void*>(peer_exchange_kernel), grid, dim3(kThreads),
                                                args, 0, static_cast<cudaStream_t>(stream))
                  : cudaLaunchKernel(reinterpret_cast<void*>(peer_exchange_kernel), grid, dim3(kThreads), args, 0,
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return SANTA_ERR_CUDA;
  }
  return SANTA_OK;
}

}  // namespace

extern "C" {

size_t santa_peer_buffer_bytes(int32_t world, size_t max_payload_bytes) {
  if (world < 1 || world > kMaxWorld || max_payload_bytes == 0) return 0;
  const size_t slot = (max_payload_bytes + 255) / 256 * 256;
  return kDataOff + 2 * (size_t)world * slot;
}

santa_status santa_peer_allgather(const santa_peer_group* group, int32_t n_local, const int32_t* ranks,
                                  const void* const* src, void* const* dst, size_t bytes, uint32_t epoch,
                                  void* stream) {
  Nvtx n_("santa_peer_allgather");
  return run(group, n_local, ranks, src, dst, bytes, epoch, 0, stream);
}

santa_status santa_peer_allreduce_f32(const santa_peer_group* group, int32_t n_local, const int32_t* ranks,
                                      const float* const* src, float* const* dst, size_t count, uint32_t epoch,
                                      void* stream) {
  Nvtx n_("santa_peer_allreduce_f32");
  if (count > (~(size_t)0) / 4) return SANTA_ERR_INVALID_ARG;
  return run(group, n_local, ranks, reinterpret_cast<const void* const*>(src), reinterpret_cast<void* const*>(dst),
             count * 4, epoch, 1, stream);
}

santa_status santa_ipc_export(const void* dev_ptr, void* handle_out, size_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return SANTA_ERR_INVALID_ARG;
  // the IPC handle names the whole allocation; the importer adds the offset of dev_ptr in it
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static const GetRange get_range = []() -> GetRange {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<GetRange>(p);
    cudaGetLastError();
    return nullptr;
  }();
  if (!get_range) return SANTA_ERR_CUDA;
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0) return SANTA_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return SANTA_ERR_CUDA;
  }
  static_assert(sizeof(h) == SANTA_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uintptr_t>(dev_ptr) - base;
  return SANTA_OK;
}

santa_status santa_ipc_import(const void* handle, size_t offset, void** dev_ptr_out, void** base_out) {
  if (!handle || !dev_ptr_out || !base_out) return SANTA_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return SANTA_ERR_CUDA;
  }
  *base_out = base;
  *dev_ptr_out = static_cast<char*>(base) + offset;
  return SANTA_OK;
}

santa_status santa_ipc_close(void* base) {
  if (!base) return SANTA_ERR_INVALID_ARG;
  if (cudaIpcCloseMemHandle(base) != cudaSuccess) {
    cudaGetLastError();
    return SANTA_ERR_CUDA;
  }
  return SANTA_OK;
}

}  // extern "C"
