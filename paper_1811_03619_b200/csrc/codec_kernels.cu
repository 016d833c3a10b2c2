// Whole-vector codec kernels and the fused gradient consumer (sm_100a).
//
//   gp_encode / gp_decode  compression.py:103-151 on one whole vector
//                          (the engine's local pre-compress, engine.py:333,
//                          and the pipe re-compress of the sum, engine.py:407)
//   gp_roundtrip           D(C(x)) without materialising the payload
//   gp_consume_update      decode slot -> fl(g / f32(p)) (engine.py:123-129)
//                          -> fl(w - fl(f32(lr) * g)) (models.py:198-204)
//
// All kernels are HBM-bound streaming passes: 8 elements per thread per
// step with 16/32-byte vector accesses, grid = a multiple of the SM count,
// grid-stride loops. quant8 needs max|x| before any code can be written,
// so it is two launches: absmax (atomicMax of float bits) then encode.
#include <cstdlib>
#include <string>

#include "../../include/pipesgd.h"
#include "codec.cuh"

using namespace gp;

void gp_set_error_string(const std::string& m);  // comm.cu: the thread's last error

namespace {

constexpr int kT = 256;
#ifndef PIPESGD_CU_ELEMS
#define PIPESGD_CU_ELEMS 8
#endif
#ifndef PIPESGD_CU_MINB
#define PIPESGD_CU_MINB 1
#endif
// fp32 elements per thread per streaming iteration, the same for every
// codec: kU<E> = max(1, 8 / E) groups of E elements (2 x fp32 groups, 1 x
// trunc16, 1 x quant8), so registers do not grow with E. Measured cold-L2
// at 4.7 M elements against 16/32 elements and the earlier 4-groups-of-any-E
// loop (profiles/r01_final/codec_kernel_variants.md): consume_update
// trunc16 19.4 -> 16.7 us, quant8 33.9 -> 19.1 us.
constexpr int kElems = PIPESGD_CU_ELEMS;
template <int E> constexpr int kU = kElems / E > 0 ? kElems / E : 1;

int cfail(int code, const std::string& m);

uint32_t grid_for(uint64_t n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  static const uint64_t per_sm = [] {
    const char* e = std::getenv("PIPESGD_CU_GRID_PER_SM");
    return (uint64_t)(e ? std::max(1, std::atoi(e)) : 8);
  }();
  const uint64_t per_block = (uint64_t)kT * std::max(kElems, 16);
  const uint64_t want = (n + per_block - 1) / per_block;
  const uint64_t cap = (uint64_t)sms * per_sm;
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, cap));
}

#define GROUP_LOOP(E) \
  for (uint64_t g0 = (uint64_t)(E) * (blockIdx.x * (uint64_t)kT + threadIdx.x); g0 < n; \
       g0 += (uint64_t)(E) * kT * gridDim.x)

// Streaming loop with kU groups per thread per iteration: every load of an
// iteration is issued before its first store (more bytes in flight per
// thread for these short HBM-bound kernels).
template <int E, typename L, typename S>
__device__ __forceinline__ void stream_groups(uint64_t n, L&& load, S&& use) {
  constexpr int U = kU<E>;
  const uint64_t stride = (uint64_t)E * kT * gridDim.x;
  for (uint64_t base = (uint64_t)E * (blockIdx.x * (uint64_t)kT + threadIdx.x); base < n; base += stride * U) {
    using T = decltype(load(base));
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * stride < n) v[u] = load(base + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * stride < n) use(base + u * stride, v[u]);
  }
}

__global__ void __launch_bounds__(kT) absmax_kernel(const float* __restrict__ x, uint64_t n,
                                                    gp_codec_status* st) {
  __shared__ uint32_t red[kT / 32];
  uint32_t m = 0;
  // 4 float4 loads in flight per thread per iteration (a load-only pass:
  // bytes in flight, not instructions, bound it); NaN bits compare above
  // +inf as unsigned, so max|x| >= 0x7F800000 flags every non-finite value
  stream_groups<16>(n, [&](uint64_t g0) { return load_fv<16>(x, g0, 0, n); },
                    [&](uint64_t, const FV<16>& v) { m = max(m, absmax_bits(v)); });
  int bad = m >= 0x7F800000u;
  m = cta_max_u32<kT>(m, red);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    atomicMax(&st->absmax_bits, m);
    if (bad) atomicOr(&st->nonfinite, 1);
  }
}

template <int C>
__device__ __forceinline__ Q8 status_scale(gp_codec_status* st) {
  Q8 q = q8_make(0.f);
  if constexpr (C == kQuant8) q = q8_make(q8_scale(__uint_as_float(*(volatile uint32_t*)&st->absmax_bits)));
  if (blockIdx.x == 0 && threadIdx.x == 0) st->scale = q.s;
  return q;
}

template <int C>
__global__ void __launch_bounds__(kT, PIPESGD_CU_MINB) encode_kernel(const float* __restrict__ x, uint64_t n,
                                                    uint8_t* payload, gp_codec_status* st) {
  constexpr int E = CodecT<C>::E;
  const Q8 q = status_scale<C>(st);
  int bad = 0;
  stream_groups<E>(n, [&](uint64_t g0) { return load_fv<E>(x, g0, 0, n); },
                   [&](uint64_t g0, const FV<E>& v) {
                     store_pay<C>(payload, g0, 0, (int)(min(n, g0 + E) - g0), encode_v<C, true, true>(v, q, bad));
                   });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->nonfinite, 1);
}

template <int C>
__global__ void __launch_bounds__(kT) decode_kernel(const uint8_t* payload, const float* scale, uint64_t n,
                                                    float* out) {
  constexpr int E = CodecT<C>::E;
  const float s = (C == kQuant8) ? *scale : 0.f;
  stream_groups<E>(n, [&](uint64_t g0) { return load_pay<C>(payload, g0, 0, (int)(min(n, g0 + E) - g0)); },
                   [&](uint64_t g0, const uint4& v) { store_fv<E>(out, g0, 0, n, decode_v<C>(v, s)); });
}

template <int C>
__global__ void __launch_bounds__(kT) roundtrip_kernel(const float* __restrict__ x, uint64_t n, float* out,
                                                       gp_codec_status* st) {
  constexpr int E = CodecT<C>::E;
  const Q8 q = status_scale<C>(st);
  int bad = 0;
  stream_groups<E>(n, [&](uint64_t g0) { return load_fv<E>(x, g0, 0, n); },
                   [&](uint64_t g0, const FV<E>& v) {
                     store_fv<E>(out, g0, 0, n, decode_v<C>(encode_v<C, true, true>(v, q, bad), q.s));
                   });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->nonfinite, 1);
}

template <int C>
__global__ void __launch_bounds__(kT, PIPESGD_CU_MINB) consume_update_kernel(float* w, const uint8_t* slot, const float* scale,
                                                            uint64_t n, float lr_val, const float* lr_dev, int p) {
  constexpr int E = CodecT<C>::E;
  const float s = (C == kQuant8) ? *scale : 0.f;
  const float lr = lr_dev ? __ldg(lr_dev) : lr_val;  // device-resident rate: graph replays with decay
  const float fp = (float)p;
  struct WG {
    FV<E> w;
    uint4 g;
  };
  stream_groups<E>(n,
                   [&](uint64_t g0) {
                     return WG{load_fv<E, false>(w, g0, 0, n), load_pay<C>(slot, g0, 0, (int)(min(n, g0 + E) - g0))};
                   },
                   [&](uint64_t g0, const WG& in) {
                     const FV<E> g = decode_v<C>(in.g, s);
                     FV<E> v = in.w;
#pragma unroll
                     for (int i = 0; i < E; ++i) {
                       const float gm = p == 1 ? g.v[i] : __fdiv_rn(g.v[i], fp);
                       v.v[i] = __fsub_rn(v.v[i], __fmul_rn(lr, gm));
                     }
                     store_fv<E>(w, g0, 0, n, v);
                   });
}

// One reduce-scatter hop on one GPU (the timing model's gamma, the
// reference calibrate()'s reduce_hop: compress(decompress(block) + grad),
// harness.py:561-568): acc = x + D(in); pass 1 (quant8) max|acc|, pass 2
// out = C(acc) with that block scale. No NVLink: the hop's compute and HBM
// share, per payload byte.
template <int C>
__global__ void __launch_bounds__(kT) hop_absmax_kernel(const float* __restrict__ x, const uint8_t* in,
                                                        const float* in_scale, uint64_t n, gp_codec_status* st) {
  constexpr int E = CodecT<C>::E;
  __shared__ uint32_t red[kT / 32];
  const float s = (C == kQuant8) ? *in_scale : 0.f;
  uint32_t m = 0;
  struct XI {
    FV<E> x;
    uint4 in;
  };
  stream_groups<E>(n, [&](uint64_t g0) { return XI{load_fv<E>(x, g0, 0, n), load_pay<C>(in, g0, 0, (int)(min(n, g0 + E) - g0))}; },
                   [&](uint64_t, const XI& v) { m = max(m, absmax_bits(add_v(v.x, decode_v<C>(v.in, s)))); });
  m = cta_max_u32<kT>(m, red);
  if (threadIdx.x == 0) atomicMax(&st->absmax_bits, m);
}

template <int C>
__global__ void __launch_bounds__(kT) hop_encode_kernel(const float* __restrict__ x, const uint8_t* in,
                                                        const float* in_scale, uint64_t n, uint8_t* out,
                                                        gp_codec_status* st) {
  constexpr int E = CodecT<C>::E;
  const float s = (C == kQuant8) ? *in_scale : 0.f;
  const Q8 q = status_scale<C>(st);
  int bad = 0;
  struct XI {
    FV<E> x;
    uint4 in;
  };
  stream_groups<E>(n, [&](uint64_t g0) { return XI{load_fv<E>(x, g0, 0, n), load_pay<C>(in, g0, 0, (int)(min(n, g0 + E) - g0))}; },
                   [&](uint64_t g0, const XI& v) {
                     store_pay<C>(out, g0, 0, (int)(min(n, g0 + E) - g0),
                                  encode_v<C, true, true>(add_v(v.x, decode_v<C>(v.in, s)), q, bad));
                   });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&st->nonfinite, 1);
}

int cfail(int code, const std::string& m) {
  gp_set_error_string(m);
  return code;
}

bool mis(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0; }

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cfail(GP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return GP_OK;
}

}  // namespace

extern "C" {

int gp_encode(int codec, const float* in, uint64_t n, void* payload, gp_codec_status* st, void* stream) {
  if (codec < 0 || codec > 2) return cfail(GP_ERR_ARG, "unknown codec");
  if (!st) return cfail(GP_ERR_ARG, "null status");
  if (n && (!in || !payload)) return cfail(GP_ERR_ARG, "null buffer");
  if (n && (mis(in) || mis(payload))) return cfail(GP_ERR_ARG, "buffers must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(st, 0, sizeof(*st), s);
  if (e != cudaSuccess) return cfail(GP_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  if (n == 0) return GP_OK;
  const uint32_t g = grid_for(n);
  auto* pl = static_cast<uint8_t*>(payload);
  if (codec == kQuant8) {
    absmax_kernel<<<g, kT, 0, s>>>(in, n, st);
    encode_kernel<kQuant8><<<g, kT, 0, s>>>(in, n, pl, st);
  } else if (codec == kTrunc16) {
    encode_kernel<kTrunc16><<<g, kT, 0, s>>>(in, n, pl, st);
  } else {
    encode_kernel<kNone><<<g, kT, 0, s>>>(in, n, pl, st);
  }
  return check_launch("encode kernel");
}

int gp_decode(int codec, const void* payload, const float* scale, uint64_t n, float* out, void* stream) {
  if (codec < 0 || codec > 2) return cfail(GP_ERR_ARG, "unknown codec");
  if (n && (!payload || !out)) return cfail(GP_ERR_ARG, "null buffer");
  if (n && codec == kQuant8 && !scale) return cfail(GP_ERR_ARG, "quant8 decode needs a scale");
  if (n && (mis(payload) || mis(out))) return cfail(GP_ERR_ARG, "buffers must be 16-byte aligned");
  if (n == 0) return GP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t g = grid_for(n);
  auto* pl = static_cast<const uint8_t*>(payload);
  if (codec == kQuant8) decode_kernel<kQuant8><<<g, kT, 0, s>>>(pl, scale, n, out);
  else if (codec == kTrunc16) decode_kernel<kTrunc16><<<g, kT, 0, s>>>(pl, scale, n, out);
  else decode_kernel<kNone><<<g, kT, 0, s>>>(pl, scale, n, out);
  return check_launch("decode kernel");
}

int gp_roundtrip(int codec, const float* in, float* out, uint64_t n, gp_codec_status* st, void* stream) {
  if (codec < 0 || codec > 2) return cfail(GP_ERR_ARG, "unknown codec");
  if (!st) return cfail(GP_ERR_ARG, "null status");
  if (n && (!in || !out)) return cfail(GP_ERR_ARG, "null buffer");
  if (n && (mis(in) || mis(out))) return cfail(GP_ERR_ARG, "buffers must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(st, 0, sizeof(*st), s);
  if (e != cudaSuccess) return cfail(GP_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  if (n == 0) return GP_OK;
  const uint32_t g = grid_for(n);
  if (codec == kQuant8) {
    absmax_kernel<<<g, kT, 0, s>>>(in, n, st);
    roundtrip_kernel<kQuant8><<<g, kT, 0, s>>>(in, n, out, st);
  } else if (codec == kTrunc16) {
    roundtrip_kernel<kTrunc16><<<g, kT, 0, s>>>(in, n, out, st);
  } else {
    roundtrip_kernel<kNone><<<g, kT, 0, s>>>(in, n, out, st);
  }
  return check_launch("roundtrip kernel");
}

static int consume_update(float* w, int codec, const void* slot, const float* scale, uint64_t n, float lr,
                          const float* lr_dev, int world, void* stream) {
  if (codec < 0 || codec > 2) return cfail(GP_ERR_ARG, "unknown codec");
  if (world < 1) return cfail(GP_ERR_ARG, "worker count must be >= 1");
  if (n && (!w || !slot)) return cfail(GP_ERR_ARG, "null buffer");
  if (n && codec == kQuant8 && !scale) return cfail(GP_ERR_ARG, "quant8 slot needs a scale");
  if (n && (mis(w) || mis(slot))) return cfail(GP_ERR_ARG, "buffers must be 16-byte aligned");
  if (n == 0) return GP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t g = grid_for(n);
  auto* pl = static_cast<const uint8_t*>(slot);
  if (codec == kQuant8) consume_update_kernel<kQuant8><<<g, kT, 0, s>>>(w, pl, scale, n, lr, lr_dev, world);
  else if (codec == kTrunc16) consume_update_kernel<kTrunc16><<<g, kT, 0, s>>>(w, pl, scale, n, lr, lr_dev, world);
  else consume_update_kernel<kNone><<<g, kT, 0, s>>>(w, pl, scale, n, lr, lr_dev, world);
  return check_launch("consume_update kernel");
}

int gp_consume_update(float* w, int codec, const void* slot, const float* scale, uint64_t n, float lr,
                      int world, void* stream) {
  return consume_update(w, codec, slot, scale, n, lr, nullptr, world, stream);
}

int gp_calib_hop(int codec, const float* x, const void* in, const float* in_scale, void* out, uint64_t n,
                 int grid, gp_codec_status* st, void* stream) {
  if (codec < 0 || codec > 2) return cfail(GP_ERR_ARG, "unknown codec");
  if (!st) return cfail(GP_ERR_ARG, "null status");
  if (n && (!x || !in || !out)) return cfail(GP_ERR_ARG, "null buffer");
  if (n && codec == kQuant8 && !in_scale) return cfail(GP_ERR_ARG, "quant8 hop needs the incoming scale");
  if (n && (mis(x) || mis(in) || mis(out))) return cfail(GP_ERR_ARG, "buffers must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(st, 0, sizeof(*st), s);
  if (e != cudaSuccess) return cfail(GP_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  if (n == 0) return GP_OK;
  const uint32_t g = grid > 0 ? (uint32_t)grid : grid_for(n);
  auto* pi = static_cast<const uint8_t*>(in);
  auto* po = static_cast<uint8_t*>(out);
  if (codec == kQuant8) {
    hop_absmax_kernel<kQuant8><<<g, kT, 0, s>>>(x, pi, in_scale, n, st);
    hop_encode_kernel<kQuant8><<<g, kT, 0, s>>>(x, pi, in_scale, n, po, st);
  } else if (codec == kTrunc16) {
    hop_encode_kernel<kTrunc16><<<g, kT, 0, s>>>(x, pi, in_scale, n, po, st);
  } else {
    hop_encode_kernel<kNone><<<g, kT, 0, s>>>(x, pi, in_scale, n, po, st);
  }
  return check_launch("hop kernel");
}

int gp_consume_update_dev(float* w, int codec, const void* slot, const float* scale, uint64_t n,
                          const float* lr, int world, void* stream) {
  if (n && !lr) return cfail(GP_ERR_ARG, "null learning-rate pointer");
  return consume_update(w, codec, slot, scale, n, 0.f, lr, world, stream);
}

}  // extern "C"
