// Calibration kernels for the paper's timing model (Eq. 5, timing.py:119-132)
// re-targeted at NVLink: beta from a peer copy (push = local load + remote
// st.global, pull = remote ld.global + local store), alpha from a flag
// ping-pong between two GPUs (one st.release.sys / ld.acquire.sys round trip
// per iteration). Reference calibrate(): harness.py:513-586.
#include <string>

#include "../../include/pipesgd.h"
#include "common.cuh"

using namespace gp;

void gp_set_error_string(const std::string& m);

namespace {

constexpr int kCT = 512;
constexpr int kCU = 8;

// Each warp streams 16-byte vectors, kCU in flight per lane.
// mode bit 0: pull (remote load, local store) instead of push.
// mode bit 1: each warp copies contiguous `chunk`-vector pieces taken from a
//             global counter (the ring kernel's access pattern) instead of
//             the grid-interleaved stride; bit 2: st.release.sys a flag after
//             every piece (the ring's publish).
__global__ void __launch_bounds__(kCT) p2p_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                       uint64_t nvec, int mode, uint64_t chunk,
                                                       unsigned long long* counter, uint64_t* flags) {
  const int pull = mode & 1;
  const uint64_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)kCT + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)kCT) >> 5;
  if (mode & 8) {
    // bit 3: CTA-aggregated publish -- every warp copies one chunk, the CTA
    // meets at a barrier, one thread issues ONE system fence and relaxed
    // flag stores for all of the CTA's chunks (instead of a release per warp)
    __shared__ uint64_t s_chunks[kCT / 32];
    for (;;) {
      uint64_t c = 0;
      if (lane == 0) c = atomicAdd(counter, 1ull);
      c = __shfl_sync(0xffffffffu, c, 0);
      const uint64_t b0 = c * chunk;
      if (b0 < nvec) {
        const uint64_t e0 = min(nvec, b0 + chunk);
        for (uint64_t base = b0; base < e0; base += 32 * kCU) {
          uint4 v[kCU];
#pragma unroll
          for (int u = 0; u < kCU; ++u) {
            const uint64_t i = base + u * 32 + lane;
            if (i < e0) v[u] = pull ? __ldcg(src + i) : __ldg(src + i);
          }
#pragma unroll
          for (int u = 0; u < kCU; ++u) {
            const uint64_t i = base + u * 32 + lane;
            if (i < e0) __stcg(dst + i, v[u]);
          }
        }
      }
      if (lane == 0) s_chunks[threadIdx.x >> 5] = b0 < nvec ? c : ~0ull;
      const int any = __syncthreads_or(b0 < nvec);
      if (!any) break;
      if (threadIdx.x == 0) {
        fence_sys();
        for (int w = 0; w < kCT / 32; ++w)
          if (s_chunks[w] != ~0ull) st_relaxed_sys(flags + s_chunks[w], 1);
      }
      __syncthreads();
    }
    return;
  }
  if (mode & 2) {
    for (;;) {
      uint64_t c = 0;
      if (lane == 0) c = atomicAdd(counter, 1ull);
      c = __shfl_sync(0xffffffffu, c, 0);
      const uint64_t b0 = c * chunk;
      if (b0 >= nvec) break;
      const uint64_t e0 = min(nvec, b0 + chunk);
      for (uint64_t base = b0; base < e0; base += 32 * kCU) {
        uint4 v[kCU];
#pragma unroll
        for (int u = 0; u < kCU; ++u) {
          const uint64_t i = base + u * 32 + lane;
          if (i < e0) v[u] = pull ? __ldcg(src + i) : __ldg(src + i);
        }
#pragma unroll
        for (int u = 0; u < kCU; ++u) {
          const uint64_t i = base + u * 32 + lane;
          if (i < e0) __stcg(dst + i, v[u]);
        }
      }
      if (mode & 4) {
        __syncwarp();
        if (lane == 0) st_release_sys(flags + c, 1);
      }
    }
    return;
  }
  for (uint64_t base = warp * 32 * kCU; base < nvec; base += nwarps * 32 * kCU) {
    uint4 v[kCU];
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
      const uint64_t i = base + u * 32 + lane;
      if (i < nvec) v[u] = pull ? __ldcg(src + i) : __ldg(src + i);
    }
#pragma unroll
    for (int u = 0; u < kCU; ++u) {
      const uint64_t i = base + u * 32 + lane;
      if (i < nvec) __stcg(dst + i, v[u]);
    }
  }
}

// One thread: `iters` rounds of (wait my flag == k, write peer flag = k).
// The initiator writes first. Flags are u64 in device memory; `mine` is
// local, `theirs` is the peer's flag mapped into this device.
__global__ void pingpong_kernel(uint64_t* mine, uint64_t* theirs, int iters, int initiator, uint64_t base,
                                unsigned long long* ns_out) {
  const uint64_t t0 = globaltimer();
  const uint64_t deadline = t0 + 10ull * 1000 * 1000 * 1000;  // never hang the box: 10 s cap
  for (int k = 1; k <= iters; ++k) {
    const uint64_t want = base + k;
    if (initiator) st_release_sys(theirs, want);
    while (ld_acquire_sys(mine) < want) {
      if (globaltimer() > deadline) {
        *ns_out = ~0ull;
        return;
      }
    }
    if (!initiator) st_release_sys(theirs, want);
  }
  *ns_out = globaltimer() - t0;
}

}  // namespace

extern "C" {

int gp_calib_p2p_copy(void* dst, const void* src, uint64_t bytes, int ctas, int pull, void* stream) {
  return gp_calib_p2p_copy_ex(dst, src, bytes, ctas, pull, 0, nullptr, nullptr, stream);
}

int gp_calib_p2p_copy_ex(void* dst, const void* src, uint64_t bytes, int ctas, int mode, uint64_t chunk_bytes,
                         void* counter, void* flags, void* stream) {
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 15u) {
    gp_set_error_string("p2p copy needs 16-byte aligned pointers and size");
    return GP_ERR_ARG;
  }
  if (ctas <= 0) ctas = 148;
  if ((mode & 10) && (!counter || chunk_bytes < 16 || ((mode & 12) && !flags))) {
    gp_set_error_string("chunked p2p copy needs a counter, chunk size and (mode 4) flags");
    return GP_ERR_ARG;
  }
  p2p_copy_kernel<<<ctas, kCT, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint4*>(dst), static_cast<const uint4*>(src), bytes / 16, mode, chunk_bytes / 16,
      static_cast<unsigned long long*>(counter), static_cast<uint64_t*>(flags));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gp_set_error_string(std::string("p2p copy launch: ") + cudaGetErrorString(e));
    return GP_ERR_CUDA;
  }
  return GP_OK;
}

int gp_calib_pingpong(void* mine, void* theirs, int iters, int initiator, uint64_t base, void* ns_out,
                      void* stream) {
  pingpong_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint64_t*>(mine), static_cast<uint64_t*>(theirs), iters, initiator, base,
      static_cast<unsigned long long*>(ns_out));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gp_set_error_string(std::string("pingpong launch: ") + cudaGetErrorString(e));
    return GP_ERR_CUDA;
  }
  return GP_OK;
}

}  // extern "C"
