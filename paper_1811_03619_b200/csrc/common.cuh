// Shared device primitives for the Pipe-SGD hot path (sm_100a).
//
// Memory-ordering helpers for cross-GPU flags (release/acquire at .sys
// scope, so NVLink peer stores become visible before the flag that
// publishes them), the device error word, and 8-element vector groups.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gp {

constexpr int kMaxRanks = 8;

enum Codec : int { kNone = 0, kTrunc16 = 1, kQuant8 = 2 };

// Error kinds latched by kernels; surfaced by the host as the reference's
// exception classes (errors.py:16-29): NONFINITE -> CodecError,
// TIMEOUT/HEADER/ABORT -> CollectiveError.
enum ErrKind : int { kErrNone = 0, kErrNonFinite = 1, kErrTimeout = 2, kErrHeader = 3, kErrBounds = 4 };
enum Phase : int { kPhRS = 0, kPhAG = 1, kPhBarrier = 2, kPhLocal = 3 };

// Device error word: one u64 so the EARLIEST failure wins via atomicMin,
// ordered by (phase order, step) like the reference, which fails at the
// first step that cannot complete. 0xFF..F = no error.
//   [63] consequence (a wait that only ended because a peer aborted: any
//        cause this rank detected itself -- timeout, header, non-finite --
//        beats every consequence)
//   [62:60] phase order (0 reduce-scatter, 1 barrier, 2 allgather, 3 local)
//   [59:53] step   [51:48] kind   [47:40] block+1   [39:32] rank   [31:0] detail
struct ErrWord {
  unsigned long long code;
  unsigned long long pad[3];
};

__host__ __device__ inline int phase_order(int phase) {
  return phase == kPhRS ? 0 : phase == kPhBarrier ? 1 : phase == kPhAG ? 2 : 3;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Record a failure; the earliest (phase, step) is kept among this rank's own
// causes (header mismatch, own timeout, non-finite); a wait that only ended
// because a peer aborted (timeout kind, detail 1) is reported only when the
// rank has no cause of its own. Steps fit 7 bits (p <= 8).
inline __device__ __noinline__ void latch_error(ErrWord* e, int kind, int phase, int step, int block,
                                         int rank, int detail) {
  const unsigned long long consequence = (kind == kErrTimeout && detail == 1) ? 1ull : 0ull;
  const unsigned long long code =
      (consequence << 63) | ((unsigned long long)(phase_order(phase) & 0x7) << 60) |
      ((unsigned long long)(step & 0x7F) << 53) |
      ((unsigned long long)(kind & 0xF) << 48) | ((unsigned long long)((block + 1) & 0xFF) << 40) |
      ((unsigned long long)(rank & 0xFF) << 32) | (unsigned long long)(uint32_t)detail;
  atomicMin(&e->code, code);
  __threadfence();
}

__device__ __forceinline__ bool nonfinite(float x) {
  return (__float_as_uint(x) & 0x7F800000u) == 0x7F800000u;
}

// Warp / CTA max of non-negative float bit patterns (uint order == float order).
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int THREADS>
__device__ __forceinline__ uint32_t cta_max_u32(uint32_t v, uint32_t* smem /*[THREADS/32]*/) {
  v = warp_max_u32(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) smem[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < THREADS / 32) ? smem[l] : 0u;
    v = warp_max_u32(v);
    if (l == 0) smem[0] = v;
  }
  __syncthreads();
  v = smem[0];
  __syncthreads();
  return v;
}

template <int THREADS>
__device__ __forceinline__ int cta_or(int v, int* smem) {
  v = __any_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) smem[threadIdx.x >> 5] = v;
  __syncthreads();
  int r = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < THREADS / 32; ++i) r |= smem[i];
    smem[0] = r;
  }
  __syncthreads();
  r = smem[0];
  __syncthreads();
  return r;
}

}  // namespace gp
