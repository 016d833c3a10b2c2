// NVLink push A/B: register stores (LDG.128 -> STG.128 to the peer, the ring's
// path) vs bulk-async copies (cp.async.bulk global -> shared, then
// cp.async.bulk shared -> peer global, i.e. TMA-style bulk moves, one elected
// lane per warp). GPU0 and GPU1 push 256 MiB to each other at the same time
// (bidirectional, like every ring phase); prints GB/s per direction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o p2p_bulk_probe tools/p2p_bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kT = 128;

__global__ void __launch_bounds__(kT) push_reg(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t nvec) {
  const uint64_t lane = threadIdx.x & 31, warp = (blockIdx.x * (uint64_t)kT + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)kT) >> 5;
  constexpr int U = 8;
  for (uint64_t base = warp * 32 * U; base < nvec; base += nw * 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + u * 32 + lane < nvec) v[u] = __ldg(src + base + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u) if (base + u * 32 + lane < nvec) __stcg(dst + base + u * 32 + lane, v[u]);
  }
}

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// each warp: S stages of `chunk` bytes; lane 0 loads a chunk into smem with a
// bulk copy (mbarrier complete_tx), then bulk-stores it to the peer
// (bulk_group), waiting for the store to have read smem before reuse
template <int S>
__global__ void __launch_bounds__(kT) push_bulk(uint8_t* dst, const uint8_t* src, uint64_t bytes, unsigned chunk) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = smem + (size_t)wl * S * (chunk + 16);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)(kT / 32) * S * (chunk + 16)) + wl * S;
  const uint64_t warp = (blockIdx.x * (uint64_t)kT + threadIdx.x) >> 5, nw = (gridDim.x * (uint64_t)kT) >> 5;
  if (lane != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  unsigned phase[S] = {};
  int k = 0;
  for (uint64_t off = warp * (uint64_t)chunk; off < bytes; off += nw * (uint64_t)chunk, k = (k + 1) % S) {
    const unsigned n = (unsigned)min((uint64_t)chunk, bytes - off);
    uint8_t* b = buf + (size_t)k * (chunk + 16);
    // the stage's previous store must have finished reading smem
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[k])), "r"(n) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(b)),
                 "l"(src + off), "r"(n), "r"(sa(&bar[k]))
                 : "memory");
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                     sa(&bar[k])),
                 "r"(phase[k])
                 : "memory");
    phase[k] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(sa(b)), "r"(n)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t bytes = 256ull << 20;
  uint8_t *a0, *b0, *a1, *b1;
  cudaSetDevice(0); cudaDeviceEnablePeerAccess(1, 0); cudaMalloc(&a0, bytes); cudaMalloc(&b0, bytes);
  cudaSetDevice(1); cudaDeviceEnablePeerAccess(0, 0); cudaMalloc(&a1, bytes); cudaMalloc(&b1, bytes);
  cudaStream_t s[2];
  cudaEvent_t e[2][2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    cudaStreamCreate(&s[d]);
    cudaEventCreate(&e[d][0]); cudaEventCreate(&e[d][1]);
  }
  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 3; ++rep) {
      for (int d = 0; d < 2; ++d) {
        cudaSetDevice(d);
        cudaEventRecord(e[d][0], s[d]);
        launch(d);
        cudaEventRecord(e[d][1], s[d]);
      }
      float ms[2];
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaEventSynchronize(e[d][1]); cudaEventElapsedTime(&ms[d], e[d][0], e[d][1]); }
      if (rep == 2) {
        const float m = ms[0] > ms[1] ? ms[0] : ms[1];
        printf("%-28s %7.3f ms  %6.1f GB/s per direction  (%s)\n", name, m, bytes / (m * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
      }
    }
  };
  for (int ctas : {148, 296, 592}) {
    char nm[64];
    snprintf(nm, sizeof nm, "register STG, %d CTAs", ctas);
    run(nm, [&](int d) {
      push_reg<<<ctas, kT, 0, s[d]>>>((uint4*)(d ? b0 : b1), (const uint4*)(d ? a1 : a0), bytes / 16);
    });
  }
  for (unsigned chunk : {4096u, 16384u}) {
    for (int ctas : {148, 296}) {
      const size_t sm = (size_t)(kT / 32) * 2 * (chunk + 16) + 64 * 8;
      cudaSetDevice(0); cudaFuncSetAttribute(push_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cudaSetDevice(1); cudaFuncSetAttribute(push_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      char nm[64];
      snprintf(nm, sizeof nm, "bulk %u B x2 stages, %d CTAs", chunk, ctas);
      run(nm, [&](int d) {
        push_bulk<2><<<ctas, kT, sm, s[d]>>>(d ? b0 : b1, d ? a1 : a0, bytes, chunk);
      });
    }
  }
  return 0;
}
