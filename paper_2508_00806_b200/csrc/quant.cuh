// Quantiser building blocks shared by the group kernels (group.cu) and the
// fused single-launch outlier-separated kernel (fused.cu).
//
// Reference: _quantize (codec.py:216-242), zeroing of flagged channels in
// compress_outlier_separated (codec.py:328-330).
#pragma once

#include "common.cuh"

namespace adc {

template <int L>
__device__ __forceinline__ uint32_t warp_max_u2(uint32_t v) {
#pragma unroll
  for (int o = 1; o < L; o <<= 1) v = __vmaxu2(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int L>
__device__ __forceinline__ uint32_t warp_min_u2(uint32_t v) {
#pragma unroll
  for (int o = 1; o < L; o <<= 1) v = __vminu2(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Zero the flagged channels of 8 consecutive elements of one row: byte j of
// f (0/1) is the flag of element j; 16-bit lane j is kept iff its flag is 0.
// Branch-free (a per-segment branch executed for whole warps anyway, ~23
// instructions per 8 elements in ncu): flags * 0xFF turns each 0/1 byte into
// 0x00/0xFF, one PRMT doubles two of them into a 16-bit-lane mask, one LOP3
// clears the lanes -- 10 instructions per 8 elements.
__device__ __forceinline__ void zero_apply8(uint32_t *w, uint2 f) {
  const uint32_t mx = f.x * 0xffu, my = f.y * 0xffu;
  w[0] &= ~__byte_perm(mx, 0u, 0x1100);
  w[1] &= ~__byte_perm(mx, 0u, 0x3322);
  w[2] &= ~__byte_perm(my, 0u, 0x1100);
  w[3] &= ~__byte_perm(my, 0u, 0x3322);
}

__device__ __forceinline__ float lo_f(uint32_t w) {
  return __low2float(*reinterpret_cast<const __half2 *>(&w));
}
__device__ __forceinline__ float hi_f(uint32_t w) {
  return __high2float(*reinterpret_cast<const __half2 *>(&w));
}

// Raw-word element access.  bf16 inputs are quantised NATIVELY: every bf16
// value with |x| >= 2^-17 is exactly representable in f16 (8-bit vs 11-bit
// mantissa), so f16(x) == x and the per-element f32->f16->f32 round trip of
// codec.py:158 is skipped.  Only groups whose scale could be affected by the
// subnormal f16 rounding of tiny values take the converting path; f16 inputs
// need no conversion at all; f32 inputs are converted to f16 on load.
template <int DT>
struct Raw {  // f16 words (F16, F32-converted)
  static constexpr bool kBf16 = false;
  template <bool KEEP>
  __device__ __forceinline__ static uint4 load8(const void *x, int64_t i) {
    return Loader<DT>::template load8<KEEP>(x, i);
  }
  __device__ __forceinline__ static float lo(uint32_t w) { return lo_f(w); }
  __device__ __forceinline__ static float hi(uint32_t w) { return hi_f(w); }
};
template <>
struct Raw<ADC_BF16> {
  static constexpr bool kBf16 = true;
  template <bool KEEP>
  __device__ __forceinline__ static uint4 load8(const void *x, int64_t i) {
    return Loader<ADC_F16>::template load8<KEEP>(x, i);  // raw 16-bit words
  }
  __device__ __forceinline__ static float lo(uint32_t w) { return __uint_as_float(w << 16); }
  __device__ __forceinline__ static float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
};

__device__ __forceinline__ uint32_t bf16_bits_to_f16_bits(uint32_t b) {
  return __half_as_ushort(__float2half_rn(__uint_as_float(b << 16)));
}

// Exact (converting) element codes for one unit: h = f16(x), float64 quotient
// as in codec.py:223-231.  Used for the rare groups / units the fast paths
// cannot decide.
template <bool BF16, int NW>
__device__ __forceinline__ void unit_codes_exact(const uint32_t *w, float s, float o, bool asym,
                                                 uint32_t *t) {
#pragma unroll
  for (int i = 0; i < 2 * NW; ++i) {
    const uint32_t raw = (w[i >> 1] >> (16 * (i & 1))) & 0xffffu;
    const uint32_t hb = BF16 ? bf16_bits_to_f16_bits(raw) : raw;
    const double h = static_cast<double>(h2f(hb));
    const double sd = s == 0.f ? 1.0 : static_cast<double>(s);
    double r = rint((asym ? h - static_cast<double>(o) : h) / sd);
    r = fmin(fmax(r, -8.0), 7.0);
    t[i] = 0x4B400008u + static_cast<uint32_t>(static_cast<int>(r));
  }
}

// Rare symmetric cases, kept out of line (the callers are hot loops and the
// instruction cache is small): a subnormal or zero scale (clip both ends),
// or a bf16 group whose maximum is so small that f16 rounding of its
// elements matters (exact converting path).
template <bool BF>
__device__ __noinline__ uint32_t sym_codes_slow(uint4 v, uint16_t s_bits, bool native) {
  using R = Raw<BF ? ADC_BF16 : ADC_F16>;
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t t[8];
  if (!BF || native) {
    const float s0 = h2f(s_bits), sc = s0 == 0.f ? 1.f : s0, inv = rcp_approx(sc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      t[2 * i] = sym_tbits_clip2(R::lo(w[i]), sc, inv);
      t[2 * i + 1] = sym_tbits_clip2(R::hi(w[i]), sc, inv);
    }
  } else {
    unit_codes_exact<BF, 4>(w, h2f(s_bits), 0.f, false, t);
  }
  return pack8_tbits(t);
}

// Symmetric int4 codes of one 8-element unit held in registers (raw words of
// the input's 16-bit format), its group spread over L aligned lanes.  Every
// lane of the warp must call (inactive lanes with act = false).  Returns the
// packed code word; s_bits / bad receive the group's scale and finiteness.
template <bool BF, int L>
__device__ __forceinline__ uint32_t sym_unit8(const uint32_t *w, bool act, uint16_t &s_bits,
                                              bool &bad) {
  using R = Raw<BF ? ADC_BF16 : ADC_F16>;
  uint32_t m = 0;
  if (act) {
#pragma unroll
    for (int i = 0; i < 4; ++i) m = __vmaxu2(m, w[i] & 0x7fff7fffu);
  }
  m = warp_max_u2<L>(m);
  const uint32_t top = max(m & 0xffffu, m >> 16);
  bool native = true;
  if (BF) {
    bad = top >= 0x4780u;     // >= 65536 rounds to f16 inf (also inf/NaN)
    native = top >= 0x3900u;  // top >= 2^-13: tiny-value rounding is code-neutral
    s_bits = sym_scale_bits(bf16_bits_to_f16_bits(top));
  } else {
    bad = top >= 0x7c00u;
    s_bits = sym_scale_bits(top);
  }
  if (!act) return 0u;
  if ((!BF || native) && s_bits >= 0x0400u) {
    uint32_t t[8];
    // normal scale: r = h/s correctly rounded (Markstein, two lanes per
    // FMUL2 / FFMA2), RNE to an integer by the magic add, upper clip to 7 on
    // the bit pattern (|h/s| < 8.004: the lower clip never binds here)
    const float sc = h2f(s_bits), inv = rcp_approx(sc);
    const uint64_t inv2 = f2_pack(inv, inv), ns2 = f2_pack(-sc, -sc), mg2 = f2_pack(kMagic8, kMagic8);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t h2 = f2_pack(R::lo(w[i]), R::hi(w[i]));
      const uint64_t r0 = f2_mul(h2, inv2);
      const uint64_t rem = f2_fma(r0, ns2, h2);
      const uint64_t r1 = f2_fma(rem, inv2, r0);
      float tl, th;
      f2_unpack(f2_add(r1, mg2), tl, th);
      t[2 * i] = min(__float_as_uint(tl), 0x4B40000Fu);
      t[2 * i + 1] = min(__float_as_uint(th), 0x4B40000Fu);
    }
    return pack8_tbits(t);
  }
  return sym_codes_slow<BF>(make_uint4(w[0], w[1], w[2], w[3]), s_bits, native);
}

}  // namespace adc
