// Back-to-back launch cost vs kernel parameter size (empty kernels, one
// stream, CUDA events around 2000 launches). Build: nvcc -O2 -gencode
// arch=compute_100a,code=sm_100a tools/launch_param_probe.cu -o gpurun_out/lpp
#include <cstdio>
#include <cuda_runtime.h>

template <int B> struct P { unsigned char b[B]; };
template <int B> __global__ void k(const __grid_constant__ P<B> p) {
  if (p.b[0] == 123 && threadIdx.x == 1000) printf("x");
}

template <int B> float run(int grid) {
  P<B> p{};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 100; ++i) k<B><<<grid, 128>>>(p);
  cudaEventRecord(a);
  for (int i = 0; i < 2000; ++i) k<B><<<grid, 128>>>(p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / 2000.f;
}

int main() {
  for (int grid : {1, 148, 592}) {
    printf("grid %4d: 64 B %.2f us | 1 KB %.2f us | 4 KB %.2f us per launch\n", grid, run<64>(grid), run<1024>(grid),
           run<4000>(grid));
  }
  return 0;
}
