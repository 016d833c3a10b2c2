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
#pragma once

#include "common.cuh"

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

// One element -> int8 code (as int). vmax==0 blocks never reach here with
// nonzero x; x==0 (either sign) always yields 0.
__device__ __forceinline__ int q8_encode(float x, const Q8& q) {
  if (q.zero) return x > 0.f ? 127 : (x < 0.f ? -127 : 0);
  const float a = __fmul_rn(fabsf(x), q.pre);
  const float y = __fmul_rn(a, q.inv);
  int k = (int)fminf(floorf(__fadd_rn(y, 0.5f)), 127.f);
  if (k >= 1 && __fmaf_rn((float)k - 0.5f, q.ss, -a) > 0.f)
    k -= 1;
  else if (k < 127 && __fmaf_rn((float)k + 0.5f, q.ss, -a) <= 0.f)
    k += 1;
  return x < 0.f ? -k : k;
}
__device__ __forceinline__ float q8_decode(int code, float s) { return __fmul_rn((float)code, s); }

// ---------------------------------------------------------------- wire groups
// A group is 8 consecutive elements starting at a global index that is a
// multiple of 8; its wire image is 32 / 16 / 8 bytes for none / trunc16 /
// quant8, so every full group moves with aligned vector accesses.

template <int C> struct Packed;
template <> struct Packed<kNone> { uint32_t w[8]; static constexpr int kWidth = 4; };
template <> struct Packed<kTrunc16> { uint32_t w[4]; static constexpr int kWidth = 2; };
template <> struct Packed<kQuant8> { uint32_t w[2]; static constexpr int kWidth = 1; };

template <int C>
__device__ __forceinline__ Packed<C> encode8(const F8& v, const Q8& q, int& bad) {
  Packed<C> p;
#pragma unroll
  for (int i = 0; i < 8; ++i) bad |= nonfinite(v.v[i]);
  if constexpr (C == kNone) {
#pragma unroll
    for (int i = 0; i < 8; ++i) p.w[i] = __float_as_uint(v.v[i]);
  } else if constexpr (C == kTrunc16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) p.w[i] = t16_encode(v.v[2 * i]) | (t16_encode(v.v[2 * i + 1]) << 16);
  } else {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      uint32_t w = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) w |= ((uint32_t)(q8_encode(v.v[4 * i + k], q) & 0xFF)) << (8 * k);
      p.w[i] = w;
    }
  }
  return p;
}

template <int C>
__device__ __forceinline__ F8 decode8(const Packed<C>& p, float s) {
  F8 v;
  if constexpr (C == kNone) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v.v[i] = __uint_as_float(p.w[i]);
  } else if constexpr (C == kTrunc16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v.v[2 * i] = t16_decode(p.w[i] & 0xFFFFu);
      v.v[2 * i + 1] = t16_decode(p.w[i] >> 16);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int code = (int)(int8_t)((p.w[i >> 2] >> (8 * (i & 3))) & 0xFF);
      v.v[i] = q8_decode(code, s);
    }
  }
  return v;
}

// Byte address of group element 0 inside a slot: rel0 = g0 - floor8(block start).
template <int C>
__device__ __forceinline__ Packed<C> load_packed(const uint8_t* slot, uint64_t rel0, int vlo, int vhi) {
  Packed<C> p;
  const uint8_t* base = slot + rel0 * Packed<C>::kWidth;
  if (vlo == 0 && vhi == 8) {
    if constexpr (C == kNone) {
      const uint4* q = reinterpret_cast<const uint4*>(base);
      uint4 a = __ldcg(q), b = __ldcg(q + 1);
      p.w[0] = a.x; p.w[1] = a.y; p.w[2] = a.z; p.w[3] = a.w;
      p.w[4] = b.x; p.w[5] = b.y; p.w[6] = b.z; p.w[7] = b.w;
    } else if constexpr (C == kTrunc16) {
      uint4 a = __ldcg(reinterpret_cast<const uint4*>(base));
      p.w[0] = a.x; p.w[1] = a.y; p.w[2] = a.z; p.w[3] = a.w;
    } else {
      uint2 a = __ldcg(reinterpret_cast<const uint2*>(base));
      p.w[0] = a.x; p.w[1] = a.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < (int)(sizeof(p.w) / 4); ++i) p.w[i] = 0;
    for (int i = vlo; i < vhi; ++i) {
      if constexpr (C == kNone) {
        p.w[i] = __ldcg(reinterpret_cast<const unsigned int*>(base) + i);
      } else if constexpr (C == kTrunc16) {
        const uint32_t h = __ldcg(reinterpret_cast<const unsigned short*>(base) + i);
        p.w[i >> 1] |= h << (16 * (i & 1));
      } else {
        const uint32_t b = (uint8_t)__ldcg(reinterpret_cast<const signed char*>(base) + i);
        p.w[i >> 2] |= b << (8 * (i & 3));
      }
    }
  }
  return p;
}

// Store (possibly to a peer GPU over NVLink) only lanes [vlo, vhi).
template <int C>
__device__ __forceinline__ void store_packed(uint8_t* slot, uint64_t rel0, int vlo, int vhi,
                                             const Packed<C>& p) {
  uint8_t* base = slot + rel0 * Packed<C>::kWidth;
  if (vlo == 0 && vhi == 8) {
    if constexpr (C == kNone) {
      uint4* q = reinterpret_cast<uint4*>(base);
      __stcg(q, make_uint4(p.w[0], p.w[1], p.w[2], p.w[3]));
      __stcg(q + 1, make_uint4(p.w[4], p.w[5], p.w[6], p.w[7]));
    } else if constexpr (C == kTrunc16) {
      __stcg(reinterpret_cast<uint4*>(base), make_uint4(p.w[0], p.w[1], p.w[2], p.w[3]));
    } else {
      __stcg(reinterpret_cast<uint2*>(base), make_uint2(p.w[0], p.w[1]));
    }
  } else {
    for (int i = vlo; i < vhi; ++i) {
      if constexpr (C == kNone) {
        reinterpret_cast<uint32_t*>(base)[i] = p.w[i];
      } else if constexpr (C == kTrunc16) {
        reinterpret_cast<uint16_t*>(base)[i] = (uint16_t)(p.w[i >> 1] >> (16 * (i & 1)));
      } else {
        base[i] = (uint8_t)(p.w[i >> 2] >> (8 * (i & 3)));
      }
    }
  }
}

__device__ __forceinline__ uint32_t absmax8_bits(const F8& v) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) m = max(m, __float_as_uint(v.v[i]) & 0x7FFFFFFFu);
  return m;
}

}  // namespace gp
