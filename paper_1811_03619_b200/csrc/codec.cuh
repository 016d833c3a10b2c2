// Bit-exact device restatement of the reference gradient codecs.
//
// Reference: /root/reference/pkg/src/gradpipe/compression.py
//   trunc16 encode  :114-124   (top halfword, RNE on the dropped half,
//                               +-inf pattern clamped to +-0x7F7F)
//   _quant_scale    :87-100    (f32(f64(vmax)/127), low 7 bits cleared,
//                               one grid step down on overshoot)
//   quant8 encode   :126-136   (half-away-from-zero of x/scale, clip 127)
//   decompress      :141-151   (identity / h<<16 / f32(code)*scale)
//
// quant8 codes are computed in fp32 without the reference's float64 divide:
// k0 = floor(|x|*(1/s) + 0.5) is within one of the exact answer
// k* = max{k : (k - 1/2)*s <= |x|}, and the sign of fmaf(k -+ 1/2, s, -|x|)
// decides the correction exactly (the residual is a multiple of the fp32
// grid of |x| and s, so a single rounding cannot flip its sign). Tiny scales
// are lifted by an exact power-of-two factor so 1/s stays finite and no
// operand is subnormal. Results equal the reference bit for bit
// (tests/test_gpu_codec.py vs tests/golden/codec_golden.npz).
//
// Wire groups: every lane moves exactly one 16-byte payload vector per step,
// i.e. E = 16 / width elements (4 fp32 / 8 trunc16 halfwords / 16 quant8
// codes), so a warp's payload access is 512 contiguous bytes — full 128-byte
// lines on NVLink and in HBM.
#pragma once

#include "common.cuh"

// Bounds-checked build (-DPIPESGD_CHECKED, libpipesgd_checked.so): a
// translation unit may define GP_ACCESS_OK(ptr, bytes, write) before including
// this header; every payload / vector access below asks it first and skips
// the access when it is refused (the hook records the violation). The
// product build compiles the hook away.
#ifndef GP_ACCESS_OK
#define GP_ACCESS_OK(ptr, bytes, write) true
#endif

namespace gp {

__device__ __forceinline__ uint32_t t16_encode(float x) {
  const uint32_t b = __float_as_uint(x);
  uint32_t hi = b >> 16;
  const uint32_t lo = b & 0xFFFFu;
  hi += (lo > 0x8000u) | ((lo == 0x8000u) & (hi & 1u));
  hi -= ((hi & 0x7FFFu) == 0x7F80u) ? 1u : 0u;
  return hi & 0xFFFFu;
}
__device__ __forceinline__ float t16_decode(uint32_t h) { return __uint_as_float(h << 16); }

// compression.py:87-100 — evaluated once per block by one thread.
__device__ __forceinline__ float q8_scale(float vmax) {
  const double v = (double)vmax;
  uint32_t bits = __float_as_uint(__double2float_rn(__ddiv_rn(v, 127.0))) & 0xFFFFFF80u;
  if (__dmul_rn((double)__uint_as_float(bits), 127.0) > v && bits >= 0x100u) bits -= 0x80u;
  return __uint_as_float(bits);
}

struct Q8 {
  float s;      // the block scale (what travels on the wire)
  float ss;     // s * pre   (exact)
  float inv;    // 1 / ss    (RN)
  float pre;    // 1 or 2^64
  int zero;     // scale == 0 (vmax tiny or 0): codes are sign(x)*127 / 0
};

__device__ __forceinline__ Q8 q8_make(float s) {
  Q8 q;
  q.s = s;
  q.zero = (s == 0.f);
  q.pre = (s < 8.673617379884035e-19f /* 2^-60 */) ? 1.8446744073709552e19f /* 2^64 */ : 1.f;
  q.ss = __fmul_rn(s, q.pre);
  q.inv = q.zero ? 0.f : __fdiv_rn(1.f, q.ss);
  return q;
}

// One element -> int8 code (as int), branch-free and without the
// quarter-rate conversion pipe (no FRND / F2I): y + 2^23 rounds y to an
// integer k0 in the low mantissa bits (RN, within one of the answer, like
// floor(y + 1/2) -- the exact residual tests below pick the right neighbour
// either way), read back as an integer by subtracting the exponent pattern
// and as an exact float by subtracting 2^23. Scale 0 (vmax tiny or 0): x/0 is
// +-inf in the reference -> +-127, and 0/0 casts to 0. x == 0 (either sign)
// always yields 0. Inputs are the block's own values, so y <= 127 * (1 +
// 2^-15); the clamp to 255 only keeps a NaN (already latched) harmless.
// GENERAL = false: the common block (scale not tiny, not zero), where the
// 2^64 lift and the zero-scale / zero-value selects are identities (a = 0
// already gives y = 0 -> code 0); the caller branches once per group.
template <bool GENERAL = true>
__device__ __forceinline__ int q8_encode(float x, const Q8& q) {
  const float a = GENERAL ? __fmul_rn(fabsf(x), q.pre) : fabsf(x);
  const float y = fminf(__fmul_rn(a, q.inv), 255.f);
  const float t = __fadd_rn(y, 8388608.f);             // 2^23 + RN(y), exact integer in the mantissa
  const float k = fminf(__fsub_rn(t, 8388608.f), 127.f);
  int c = min((int)(__float_as_uint(t) - 0x4B000000u), 127);
  const float r_lo = __fmaf_rn(__fsub_rn(k, 0.5f), q.ss, -a);  // > 0 : k too large
  const float r_hi = __fmaf_rn(__fadd_rn(k, 0.5f), q.ss, -a);  // <= 0: k too small
  c += ((c < 127) & (r_hi <= 0.f)) - ((c >= 1) & (r_lo > 0.f));
  if constexpr (GENERAL) {
    c = q.zero ? 127 : c;
    c = (a == 0.f) ? 0 : c;
  }
  return (x < 0.f) ? -c : c;
}
// code -> exact float without I2F: the byte c + 128 under the exponent of
// 2^23 is 2^23 + 128 + c; subtracting 2^23 + 128 is exact (and gives +0 for
// c = 0, like the reference's f32(0) * scale)
__device__ __forceinline__ float q8_code_float(int c) {
  return __fsub_rn(__uint_as_float(0x4B000000u + (uint32_t)(c + 128)), 8388736.f);
}
__device__ __forceinline__ float q8_decode(int code, float s) { return __fmul_rn(q8_code_float(code), s); }

// ----------------------------------------------------------- wire groups

template <int C> struct CodecT;
template <> struct CodecT<kNone> { static constexpr int W = 4, E = 4; };
template <> struct CodecT<kTrunc16> { static constexpr int W = 2, E = 8; };
template <> struct CodecT<kQuant8> { static constexpr int W = 1, E = 16; };

template <int E>
struct FV {
  float v[E];
};

__device__ __forceinline__ uint32_t wget(const uint4& p, int i) {
  return i == 0 ? p.x : i == 1 ? p.y : i == 2 ? p.z : p.w;
}

// CHECK = false where the caller has already established finiteness (the
// quant8 ring: pass A's block max covers every value pass B encodes).
// FAST = true branches once per group to the common-block quant8 encoder
// (q8_encode<false>); the ring keeps the single path (its 128-register
// budget has no room for both).
template <int C, bool CHECK = true, bool FAST = false>
__device__ __forceinline__ uint4 encode_v(const FV<CodecT<C>::E>& v, const Q8& q, int& bad) {
  constexpr int E = CodecT<C>::E;
  uint32_t w[4];
  if constexpr (CHECK) {
#pragma unroll
    for (int i = 0; i < E; ++i) bad |= nonfinite(v.v[i]);
  }
  if constexpr (C == kNone) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __float_as_uint(v.v[i]);
  } else if constexpr (C == kTrunc16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = t16_encode(v.v[2 * i]) | (t16_encode(v.v[2 * i + 1]) << 16);
  } else {
    auto pack = [&](auto enc) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t c0 = (uint32_t)enc(v.v[4 * i]), c1 = (uint32_t)enc(v.v[4 * i + 1]);
        const uint32_t c2 = (uint32_t)enc(v.v[4 * i + 2]), c3 = (uint32_t)enc(v.v[4 * i + 3]);
        w[i] = __byte_perm(__byte_perm(c0, c1, 0x0040u), __byte_perm(c2, c3, 0x0040u), 0x5410u);  // bytes c0..c3
      }
    };
    if (FAST && q.pre == 1.f && !q.zero) pack([&](float x) { return q8_encode<false>(x, q); });
    else pack([&](float x) { return q8_encode<true>(x, q); });
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <int C>
__device__ __forceinline__ FV<CodecT<C>::E> decode_v(const uint4& p, float s) {
  FV<CodecT<C>::E> v;
  const uint32_t w[4] = {p.x, p.y, p.z, p.w};
  if constexpr (C == kNone) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v.v[i] = __uint_as_float(w[i]);
  } else if constexpr (C == kTrunc16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v.v[2 * i] = t16_decode(w[i] & 0xFFFFu);
      v.v[2 * i + 1] = t16_decode(w[i] >> 16);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // byte k of a word XOR 0x80 is code + 128; PRMT places it under the
      // exponent pattern of 2^23 (0x4B0000xx), one FADD makes it the code
      const uint32_t wx = w[j] ^ 0x80808080u;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        v.v[4 * j + k] = __fmul_rn(__fsub_rn(__uint_as_float(__byte_perm(wx, 0x4B000000u, 0x7440u | k)), 8388736.f), s);
    }
  }
  return v;
}

// Partial groups (at most two per block and chunk edge) take out-of-line
// element-wise paths: inlined at every load / store site they were a large
// share of the ring kernels' instruction bytes, which small calls fetch cold.
template <int E, bool NC>
__device__ __noinline__ FV<E> load_fv_edge(const float* x, uint64_t g0, uint64_t lo, uint64_t hi) {
  FV<E> r;
  for (int i = 0; i < E; ++i)
    r.v[i] = (g0 + i >= lo && g0 + i < hi && GP_ACCESS_OK(x + g0 + i, 4, false))
                 ? (NC ? __ldg(x + g0 + i) : __ldcg(x + g0 + i)) : 0.f;
  return r;
}

// fp32 values x[g0 .. g0+E) restricted to [lo, hi); outside lanes read 0.
// NC=true uses the read-only path (inputs not written by this launch).
template <int E, bool NC = true>
__device__ __forceinline__ FV<E> load_fv(const float* x, uint64_t g0, uint64_t lo, uint64_t hi) {
  FV<E> r;
  if (lo <= g0 && g0 + E <= hi) {
    const float4* p = reinterpret_cast<const float4*>(x + g0);
    if (!GP_ACCESS_OK(p, 4 * E, false)) {
#pragma unroll
      for (int i = 0; i < E; ++i) r.v[i] = 0.f;
      return r;
    }
#pragma unroll
    for (int k = 0; k < E / 4; ++k) {
      const float4 a = NC ? __ldg(p + k) : __ldcg(p + k);
      r.v[4 * k] = a.x; r.v[4 * k + 1] = a.y; r.v[4 * k + 2] = a.z; r.v[4 * k + 3] = a.w;
    }
  } else {
    r = load_fv_edge<E, NC>(x, g0, lo, hi);
  }
  return r;
}

// L2 eviction-priority policies (createpolicy) for streams read twice: the
// first read marks lines evict_last so the second read finds them in the
// 126 MB L2; the second read marks them evict_first (their last use).
#ifndef PIPESGD_L2_KEEP
#define PIPESGD_L2_KEEP 1  // 1: evict_last, 2: evict_normal, 0: evict_first (A/B knob)
#endif
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
#if PIPESGD_L2_KEEP == 1
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#elif PIPESGD_L2_KEEP == 2
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldg_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ldcg_hint(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// load_fv of a read-only input with an L2 policy (edges take the plain path)
template <int E>
__device__ __forceinline__ FV<E> load_fv_pol(const float* x, uint64_t g0, uint64_t lo, uint64_t hi, uint64_t pol) {
  if (!(lo <= g0 && g0 + E <= hi)) return load_fv<E>(x, g0, lo, hi);
  FV<E> r;
  const float4* p = reinterpret_cast<const float4*>(x + g0);
  if (!GP_ACCESS_OK(p, 4 * E, false)) return load_fv<E>(x, g0, 1, 0);  // refused: zeros
#pragma unroll
  for (int k = 0; k < E / 4; ++k) {
    const float4 a = ldg_hint(p + k, pol);
    r.v[4 * k] = a.x; r.v[4 * k + 1] = a.y; r.v[4 * k + 2] = a.z; r.v[4 * k + 3] = a.w;
  }
  return r;
}

template <int E>
__device__ __noinline__ void store_fv_edge(float* x, uint64_t g0, uint64_t lo, uint64_t hi, const FV<E> r) {
  for (int i = 0; i < E; ++i)
    if (g0 + i >= lo && g0 + i < hi && GP_ACCESS_OK(x + g0 + i, 4, true)) x[g0 + i] = r.v[i];
}

template <int E>
__device__ __forceinline__ void store_fv(float* x, uint64_t g0, uint64_t lo, uint64_t hi, const FV<E>& r) {
  if (lo <= g0 && g0 + E <= hi) {
    float4* p = reinterpret_cast<float4*>(x + g0);
    if (!GP_ACCESS_OK(p, 4 * E, true)) return;
#pragma unroll
    for (int k = 0; k < E / 4; ++k) p[k] = make_float4(r.v[4 * k], r.v[4 * k + 1], r.v[4 * k + 2], r.v[4 * k + 3]);
  } else {
    store_fv_edge<E>(x, g0, lo, hi, r);
  }
}

// Payload vector of the group whose first element is `rel0` elements past
// the slot origin; only elements [vlo, vhi) of the group exist.
template <int C>
__device__ __noinline__ uint4 load_pay_edge(const uint8_t* base, int vlo, int vhi) {
  constexpr int W = CodecT<C>::W;
  uint32_t w[4] = {0, 0, 0, 0};
  for (int i = vlo; i < vhi; ++i) {
    uint32_t e;
    if constexpr (W == 4) e = __ldcg(reinterpret_cast<const unsigned int*>(base) + i);
    else if constexpr (W == 2) e = __ldcg(reinterpret_cast<const unsigned short*>(base) + i);
    else e = (uint8_t)__ldcg(reinterpret_cast<const signed char*>(base) + i);
    const int bit = (i * W * 8) & 31;
    w[(i * W) >> 2] |= e << bit;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <int C>
__device__ __forceinline__ uint4 load_pay(const uint8_t* slot, uint64_t rel0, int vlo, int vhi) {
  constexpr int E = CodecT<C>::E, W = CodecT<C>::W;
  const uint8_t* base = slot + rel0 * W;
  if (!GP_ACCESS_OK(base + vlo * W, (vhi - vlo) * W, false)) return make_uint4(0, 0, 0, 0);
  if (vlo == 0 && vhi == E) return __ldcg(reinterpret_cast<const uint4*>(base));
  return load_pay_edge<C>(base, vlo, vhi);
}

template <int C>
__device__ __forceinline__ uint4 load_pay_pol(const uint8_t* slot, uint64_t rel0, int vlo, int vhi, uint64_t pol) {
  constexpr int E = CodecT<C>::E, W = CodecT<C>::W;
  if (vlo == 0 && vhi == E && GP_ACCESS_OK(slot + rel0 * W, 16, false))
    return ldcg_hint(reinterpret_cast<const uint4*>(slot + rel0 * W), pol);
  return load_pay<C>(slot, rel0, vlo, vhi);
}

template <int C>
__device__ __noinline__ void store_pay_edge(uint8_t* base, int vlo, int vhi, const uint4 p) {
  constexpr int W = CodecT<C>::W;
  for (int i = vlo; i < vhi; ++i) {
    const uint32_t word = wget(p, (i * W) >> 2);
    const int bit = (i * W * 8) & 31;
    if constexpr (W == 4) reinterpret_cast<uint32_t*>(base)[i] = word;
    else if constexpr (W == 2) reinterpret_cast<uint16_t*>(base)[i] = (uint16_t)(word >> bit);
    else base[i] = (uint8_t)(word >> bit);
  }
}

template <int C>
__device__ __forceinline__ void store_pay(uint8_t* slot, uint64_t rel0, int vlo, int vhi, const uint4& p) {
  constexpr int E = CodecT<C>::E, W = CodecT<C>::W;
  uint8_t* base = slot + rel0 * W;
  if (!GP_ACCESS_OK(base + vlo * W, (vhi - vlo) * W, true)) return;
  if (vlo == 0 && vhi == E) {
    __stcg(reinterpret_cast<uint4*>(base), p);
    return;
  }
  store_pay_edge<C>(base, vlo, vhi, p);
}

template <int E>
__device__ __forceinline__ uint32_t absmax_bits(const FV<E>& v) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < E; ++i) m = max(m, __float_as_uint(v.v[i]) & 0x7FFFFFFFu);
  return m;
}

template <int E>
__device__ __forceinline__ FV<E> add_v(const FV<E>& a, const FV<E>& b) {
  FV<E> r;
#pragma unroll
  for (int i = 0; i < E; ++i) r.v[i] = __fadd_rn(a.v[i], b.v[i]);
  return r;
}

}  // namespace gp
