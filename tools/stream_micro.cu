// Micro-benchmark for the ring's streaming passes (quant8 pass A shape):
// every warp streams its own contiguous chunk of x (fp32) and of an inbox
// (1 B/elem), decodes, adds and reduces max|sum|. Strategies:
//   reg<U>  : U 16-element groups per lane in registers per batch (the ring today: U = 1)
//   bulk<S> : an S-stage per-warp shared-memory ring filled by cp.async.bulk
//             (TMA bulk copies, mbarrier complete_tx), lanes read smem
// Cold data: NB rotating buffer sets larger than L2. Prints GB/s of reads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_micro tools/stream_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kThreads = 128, kWarps = 4;
constexpr int E = 16;         // elements per lane group (16 quant8 codes = 16 B)
constexpr int BATCH = 32 * E; // 512 elements per warp batch

__device__ __forceinline__ float dec(uint32_t w, int k, float s) {
  return __fmul_rn(__fsub_rn(__uint_as_float(__byte_perm(w ^ 0x80808080u, 0x4B000000u, 0x7440u | k)), 8388736.f), s);
}

template <int U>
__global__ void __launch_bounds__(kThreads, 4) reg_kernel(const float* __restrict__ x, const uint8_t* __restrict__ in,
                                                            uint64_t n, uint64_t chunk, unsigned* out) {
  const uint64_t wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const uint64_t lo = wid * chunk, hi = min(n, lo + chunk);
  uint32_t m = 0;
  for (uint64_t b0 = lo; b0 < hi; b0 += (uint64_t)BATCH * U) {
    float4 xv[U][4];
    uint4 iv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = b0 + (uint64_t)(u * 32 + lane) * E;
      if (g < hi) {
        const float4* p = reinterpret_cast<const float4*>(x + g);
#pragma unroll
        for (int k = 0; k < 4; ++k) xv[u][k] = __ldg(p + k);
        iv[u] = __ldcg(reinterpret_cast<const uint4*>(in + g));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = b0 + (uint64_t)(u * 32 + lane) * E;
      if (g < hi) {
        const uint32_t w[4] = {iv[u].x, iv[u].y, iv[u].z, iv[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float a[4] = {xv[u][k].x, xv[u][k].y, xv[u][k].z, xv[u][k].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) m = max(m, __float_as_uint(__fadd_rn(a[j], dec(w[k], j, 0.01f))) & 0x7FFFFFFFu);
        }
      }
    }
  }
  if (m == 0x7F7FFFFEu) atomicMax(out, m);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

template <int S>
__global__ void __launch_bounds__(kThreads, 4) bulk_kernel(const float* __restrict__ x, const uint8_t* __restrict__ in,
                                                             uint64_t n, uint64_t chunk, unsigned* out) {
  // per warp: S stages x (2 KB x + 512 B inbox) + S mbarriers
  extern __shared__ __align__(128) uint8_t smem[];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* base = smem + (size_t)wl * S * (BATCH * 5 + 16);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)S * BATCH * 5);
  const uint64_t wid = blockIdx.x * kWarps + wl;
  const uint64_t lo = wid * chunk, hi = min(n, lo + chunk);
  const uint64_t nb = hi > lo ? (hi - lo + BATCH - 1) / BATCH : 0;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](uint64_t b) {
    const int s = (int)(b % S);
    const uint64_t g = lo + b * BATCH;
    const unsigned ne = (unsigned)min((uint64_t)BATCH, hi - g);
    mbar_expect(&bars[s], ne * 5);
    bulk_g2s(base + (size_t)s * BATCH * 5, x + g, ne * 4, &bars[s]);
    bulk_g2s(base + (size_t)s * BATCH * 5 + BATCH * 4, in + g, ne, &bars[s]);
  };
  if (lane == 0)
    for (uint64_t b = 0; b < min((uint64_t)S, nb); ++b) issue(b);
  uint32_t m = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    const int s = (int)(b % S);
    mbar_wait(&bars[s], (unsigned)((b / S) & 1));
    const uint64_t g0 = lo + b * BATCH + (uint64_t)lane * E;
    if (g0 < hi) {
      const float4* xs = reinterpret_cast<const float4*>(base + (size_t)s * BATCH * 5) + lane * 4;
      const uint4 iv = reinterpret_cast<const uint4*>(base + (size_t)s * BATCH * 5 + BATCH * 4)[lane];
      const uint32_t w[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 v = xs[k];
        const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) m = max(m, __float_as_uint(__fadd_rn(a[j], dec(w[k], j, 0.01f))) & 0x7FFFFFFFu);
      }
    }
    __syncwarp();
    if (lane == 0 && b + S < nb) issue(b + S);
  }
  if (m == 0x7F7FFFFEu) atomicMax(out, m);
}

int main() {
  const uint64_t n = 15275008;  // ~one C3 block at p = 4 (multiple of 512: whole bulk copies)
  const int NB = 4;             // rotating sets: 4 x (61 + 15) MB > 126 MB L2
  float* x[NB];
  uint8_t* in[NB];
  for (int i = 0; i < NB; ++i) {
    cudaMalloc(&x[i], n * 4 + 4096);
    cudaMalloc(&in[i], n + 4096);
    cudaMemset(x[i], 0, n * 4);
    cudaMemset(in[i], 0, n);
  }
  unsigned* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int ctas : {sms, 2 * sms, 4 * sms}) {
    const uint64_t warps = (uint64_t)ctas * kWarps;
    const uint64_t chunk = ((n + warps - 1) / warps + BATCH - 1) / BATCH * BATCH;
    auto run = [&](const char* name, auto launch) {
      for (int w = 0; w < 3; ++w) launch(x[w % NB], in[w % NB]);
      cudaEventRecord(a);
      const int it = 40;
      for (int i = 0; i < it; ++i) launch(x[i % NB], in[i % NB]);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("ctas=%4d %-10s %7.2f us  %7.1f GB/s  (%s)\n", ctas, name, ms * 1e3 / it, 5.0 * n / (ms * 1e-3 / it) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    };
    run("reg<1>", [&](float* xx, uint8_t* ii) { reg_kernel<1><<<ctas, kThreads>>>(xx, ii, n, chunk, out); });
    run("reg<2>", [&](float* xx, uint8_t* ii) { reg_kernel<2><<<ctas, kThreads>>>(xx, ii, n, chunk, out); });
    run("reg<4>", [&](float* xx, uint8_t* ii) { reg_kernel<4><<<ctas, kThreads>>>(xx, ii, n, chunk, out); });
    for (int S : {2, 4, 8}) {
      const size_t sm = (size_t)kWarps * S * (BATCH * 5 + 16);
      char nm[32];
      snprintf(nm, sizeof nm, "bulk<%d>", S);
      if (S == 2) {
        cudaFuncSetAttribute(bulk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        run(nm, [&](float* xx, uint8_t* ii) { bulk_kernel<2><<<ctas, kThreads, sm>>>(xx, ii, n, chunk, out); });
      } else if (S == 4) {
        cudaFuncSetAttribute(bulk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        run(nm, [&](float* xx, uint8_t* ii) { bulk_kernel<4><<<ctas, kThreads, sm>>>(xx, ii, n, chunk, out); });
      } else {
        cudaFuncSetAttribute(bulk_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        run(nm, [&](float* xx, uint8_t* ii) { bulk_kernel<8><<<ctas, kThreads, sm>>>(xx, ii, n, chunk, out); });
      }
    }
  }
  return 0;
}
