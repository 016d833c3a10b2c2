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
enum ErrKind : int { kErrNone = 0, kErrNonFinite = 1, kErrTimeout = 2, kErrHeader = 3 };
enum Phase : int { kPhRS = 0, kPhAG = 1, kPhBarrier = 2, kPhLocal = 3 };

struct ErrWord {
  int kind;
  int phase;
  int step;
  int block;
  int rank;
  int detail;
  int pad[2];
};

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

// Record the first error only (later ones are consequences).
__device__ __forceinline__ void latch_error(ErrWord* e, int kind, int phase, int step, int block,
                                            int rank, int detail) {
  if (atomicCAS(&e->kind, 0, kind) == 0) {
    e->phase = phase;
    e->step = step;
    e->block = block;
    e->rank = rank;
    e->detail = detail;
    __threadfence();
  }
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
