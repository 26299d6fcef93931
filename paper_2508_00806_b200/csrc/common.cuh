// Device helpers shared by the compressor kernels (sm_100a).
//
// Numeric contract: SURVEY.md Appendix A, restating codec.py:156-286.
//  * every input element is cast to float16 RNE first (codec.py:158);
//  * scales / offsets are float16 values computed as f16(f64 expression);
//  * codes are rint-half-even of the float64 quotient, clipped to [-8, 7];
//  * dequantisation is one rounding of code*s (+o) to float32.
// The helpers below reproduce those float64 results with float32 arithmetic
// where that is provably exact, and fall back to float64 per element only on
// exact half-integer quotients of the asymmetric scheme (Appendix A.5).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/adacc.h"

namespace adc {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// loads: 8 consecutive elements -> 8 float16 (as 4 x half2 packed in uint4)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream16(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Keeps the line in L2 for a second pass of the same kernel sequence
// (evict_last cache policy; the plain .L2::evict_last qualifier is only legal
// on 256-bit loads).
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_keep16(const void *p) {
  uint4 r;
  asm volatile(
      "{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], pol;\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream16(void *p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w));
}

__device__ __forceinline__ uint32_t f32x2_to_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);  // F2FP.F16.F32.PACK_AB, RNE
  return *reinterpret_cast<uint32_t *>(&h);
}

// bf16 pair (packed in one u32) -> f16 pair.  bf16 -> f32 is exact, so the
// only rounding is the f32 -> f16 RNE one, as numpy's astype(float16) of the
// float32 value would do.
__device__ __forceinline__ uint32_t bf2_to_h2(uint32_t u) {
  return f32x2_to_h2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}

template <int DT>
struct Loader;

template <>
struct Loader<ADC_F16> {
  static constexpr int kBytes = 2;
  template <bool KEEP>
  __device__ __forceinline__ static uint4 load8(const void *x, int64_t i) {
    const char *p = static_cast<const char *>(x) + i * 2;
    return KEEP ? ld_keep16(p) : ld_stream16(p);
  }
  __device__ __forceinline__ static uint16_t load1(const void *x, int64_t i) {
    return static_cast<const uint16_t *>(x)[i];
  }
};

template <>
struct Loader<ADC_BF16> {
  static constexpr int kBytes = 2;
  template <bool KEEP>
  __device__ __forceinline__ static uint4 load8(const void *x, int64_t i) {
    const char *p = static_cast<const char *>(x) + i * 2;
    uint4 v = KEEP ? ld_keep16(p) : ld_stream16(p);
    return make_uint4(bf2_to_h2(v.x), bf2_to_h2(v.y), bf2_to_h2(v.z), bf2_to_h2(v.w));
  }
  __device__ __forceinline__ static uint16_t load1(const void *x, int64_t i) {
    uint32_t u = static_cast<const uint16_t *>(x)[i];
    return __half_as_ushort(__float2half_rn(__uint_as_float(u << 16)));
  }
};

template <>
struct Loader<ADC_F32> {
  static constexpr int kBytes = 4;
  template <bool KEEP>
  __device__ __forceinline__ static uint4 load8(const void *x, int64_t i) {
    const char *p = static_cast<const char *>(x) + i * 4;
    uint4 a = KEEP ? ld_keep16(p) : ld_stream16(p);
    uint4 b = KEEP ? ld_keep16(p + 16) : ld_stream16(p + 16);
    return make_uint4(f32x2_to_h2(__uint_as_float(a.x), __uint_as_float(a.y)),
                      f32x2_to_h2(__uint_as_float(a.z), __uint_as_float(a.w)),
                      f32x2_to_h2(__uint_as_float(b.x), __uint_as_float(b.y)),
                      f32x2_to_h2(__uint_as_float(b.z), __uint_as_float(b.w)));
  }
  __device__ __forceinline__ static uint16_t load1(const void *x, int64_t i) {
    return __half_as_ushort(__float2half_rn(static_cast<const float *>(x)[i]));
  }
};

// ---------------------------------------------------------------------------
// float16 bit tricks
// ---------------------------------------------------------------------------
// |h| as an integer orders like the magnitude for finite f16; >= 0x7c00 means
// inf/NaN, so one integer max gives both the group abs-max and the finiteness
// check of codec.py:167-170.
__device__ __forceinline__ uint32_t absmax8(uint4 h) {
  uint32_t m = __vmaxu2(h.x & 0x7fff7fffu, h.y & 0x7fff7fffu);
  m = __vmaxu2(m, h.z & 0x7fff7fffu);
  m = __vmaxu2(m, h.w & 0x7fff7fffu);
  return m;  // two u16 lanes
}

// Monotone unsigned key of an f16 bit pattern (-0 sorts just below +0).
__device__ __forceinline__ uint32_t f16_key(uint32_t b) {
  return (b & 0x8000u) ? (~b & 0xffffu) : (b | 0x8000u);
}
__device__ __forceinline__ uint32_t f16_unkey(uint32_t k) {
  return (k & 0x8000u) ? (k & 0x7fffu) : (~k & 0xffffu);
}
// Same on both lanes of a packed pair.
__device__ __forceinline__ uint32_t f16_key2(uint32_t b) {
  uint32_t neg = ((b >> 15) & 0x00010001u) * 0xffffu;  // lane mask of negative lanes
  return (b ^ (neg | 0x80008000u));
}

__device__ __forceinline__ uint32_t hmax2_nan(uint32_t a, uint32_t b) {
  __half2 r = __hmax2_nan(*reinterpret_cast<__half2 *>(&a), *reinterpret_cast<__half2 *>(&b));
  return *reinterpret_cast<uint32_t *>(&r);
}
__device__ __forceinline__ uint32_t hmin2_nan(uint32_t a, uint32_t b) {
  __half2 r = __hmin2_nan(*reinterpret_cast<__half2 *>(&a), *reinterpret_cast<__half2 *>(&b));
  return *reinterpret_cast<uint32_t *>(&r);
}

__device__ __forceinline__ float h2f(uint32_t bits16) {
  return __half2float(__ushort_as_half(static_cast<uint16_t>(bits16)));
}

// codec.py:192-196: f16(raw) with a 2^-24 floor when a non-zero raw underflows.
__device__ __forceinline__ uint16_t store_scale_f32(float raw) {
  uint16_t s = __half_as_ushort(__float2half_rn(raw));
  if ((s & 0x7fffu) == 0 && raw > 0.f) s = 0x0001u;
  return s;
}
__device__ __forceinline__ uint16_t store_scale_f64(double raw) {
  uint16_t s = __half_as_ushort(__double2half(raw));  // cvt.rn.f16.f64, one rounding
  if ((s & 0x7fffu) == 0 && raw > 0.0) s = 0x0001u;
  return s;
}

// Symmetric scale from the group abs-max bits: top/8 is exact in f32, so the
// single f32->f16 rounding equals the reference's f64->f16 one.
__device__ __forceinline__ uint16_t sym_scale_bits(uint32_t top_bits) {
  return store_scale_f32(h2f(top_bits) * 0.125f);
}

// Asymmetric offset / scale from the group hi / lo (f16 bits), in float64
// exactly as codec.py:219-222 (hi+lo and hi-lo are exact in f64).
__device__ __forceinline__ void asym_params(uint32_t hi_bits, uint32_t lo_bits, uint16_t &off,
                                            uint16_t &scl) {
  double hi = static_cast<double>(h2f(hi_bits));
  double lo = static_cast<double>(h2f(lo_bits));
  off = __half_as_ushort(__double2half((hi + lo) * 0.5));
  scl = store_scale_f64((hi - lo) * 0.0625);
}

// Per-group quantisation constants.
struct QParams {
  float s;    // divisor: the stored scale, or 1 when it is zero (codec.py:229-230)
  float inv;  // RN(1/s)
  float o;    // offset (0 for symmetric)
};

// MUFU.RCP, ~1 ulp.  A correctly rounded reciprocal is not needed: the
// symmetric path refines the quotient with one Markstein step (exact on ties,
// within 1 ulp elsewhere), the asymmetric path widens its near-tie window.
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ QParams make_qparams(uint16_t s_bits, uint16_t o_bits) {
  QParams q;
  float s = h2f(s_bits);
  q.s = (s == 0.f) ? 1.f : s;
  q.inv = rcp_approx(q.s);
  q.o = h2f(o_bits);
  return q;
}

// Packed f32x2 arithmetic (sm_100: FFMA2 / FADD2, two lanes per instruction).
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds to int, RNE
constexpr float kMagic8 = 12582920.0f;  // kMagic + 8: low nibble of the sum = code + 8

// Symmetric code of one element as an int in [-8, 7].
// r1 is the correctly rounded f32 quotient h/s (Markstein: r0 = h*inv,
// residual exact by FMA, one correction).  Symmetric quotients are either
// exact half-integers (then r1 is exact and the RNE add ties to even) or at
// least 2^-12 away from one (Appendix A.5), so this equals rint(f64(h)/s).
__device__ __forceinline__ int sym_code(float h, const QParams &q) {
  float r0 = h * q.inv;
  float rem = fmaf(-r0, q.s, h);
  float r1 = fmaf(rem, q.inv, r0);
  r1 = fminf(fmaxf(r1, -8.f), 7.f);
  return __float_as_int(r1 + kMagic) - 0x4B400000;
}

// Asymmetric code.  d = f32(h - o) can round (tiny h against a large offset:
// the Appendix A.5 KAT), so exactness is not available in f32.  Instead:
// r = f32(d * inv) (inv = MUFU.RCP, ~1 ulp) is within ~4 ulp, i.e. < 2^-18.8
// absolute for |r| <= 9, of the exact quotient (h - o)/s.  If r is farther
// than 2^-17 from every
// half-integer, rint(r) equals the reference's rint of the float64 quotient;
// otherwise (exact ties and near-ties, ~1e-5 of random elements) the code is
// recomputed exactly in float64 exactly as codec.py:223-231 does.
static __device__ __noinline__ int asym_code_f64(float h, const QParams &q) {
  double d = static_cast<double>(h) - static_cast<double>(q.o);
  double r = rint(d / static_cast<double>(q.s));
  r = fmin(fmax(r, -8.0), 7.0);
  return static_cast<int>(r);
}

__device__ __forceinline__ int asym_code(float h, const QParams &q) {
  const float d = h - q.o;
  const float r = fminf(fmaxf(d * q.inv, -8.f), 7.f);
  const float t = r + kMagic;
  if (fabsf(r - (t - kMagic)) > 0.5f - 0x1p-17f) return asym_code_f64(h, q);
  return __float_as_int(t) - 0x4B400000;
}

template <bool ASYM>
__device__ __forceinline__ int quant_code(float h, const QParams &q) {
  if (ASYM) return asym_code(h, q);
  return sym_code(h, q);
}

// Quantise 8 f16 values (packed) and pack 8 nibbles into one u32, element 0
// in the lowest nibble (codec.py:199-203).
template <bool ASYM>
__device__ __forceinline__ uint32_t quant_pack8(uint4 h, const QParams &q) {
  uint32_t w[4] = {h.x, h.y, h.z, h.w};
  uint32_t out = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int c0 = quant_code<ASYM>(h2f(w[j] & 0xffffu), q);
    int c1 = quant_code<ASYM>(h2f(w[j] >> 16), q);
    out |= (static_cast<uint32_t>(c0) & 0xfu) << (8 * j);
    out |= (static_cast<uint32_t>(c1) & 0xfu) << (8 * j + 4);
  }
  return out;
}

// ---- 16-elements-per-lane fast path helpers -------------------------------
// "t-bits": the f32 bit pattern of r + kMagic8, whose low nibble is code + 8
// and whose bits 4..21 are zero; packing works on these directly.
//
// Symmetric, normal scale (s >= 2^-14): |h/s| <= 8/(1 - 2^-11) < 8.004, so
// rint never goes below -8 and only the upper clip is needed.
__device__ __forceinline__ uint32_t sym_tbits(float h, float s, float inv) {
  const float r0 = h * inv;
  const float rem = fmaf(-r0, s, h);
  const float r1 = fminf(fmaf(rem, inv, r0), 7.f);
  return __float_as_uint(r1 + kMagic8);
}
// Subnormal (or zero -> 1) scale: the f16 rounding of top/8 can be coarse,
// clip both ends (codec.py:231).
__device__ __forceinline__ uint32_t sym_tbits_clip2(float h, float s, float inv) {
  const float r0 = h * inv;
  const float rem = fmaf(-r0, s, h);
  const float r1 = fminf(fmaxf(fmaf(rem, inv, r0), -8.f), 7.f);
  return __float_as_uint(r1 + kMagic8);
}
__device__ __forceinline__ uint32_t asym_tbits(float h, const QParams &q) {
  const float d = h - q.o;
  const float r = fminf(fmaxf(d * q.inv, -8.f), 7.f);
  const float t = r + kMagic8;
  if (fabsf(r - (t - kMagic8)) > 0.5f - 0x1p-17f)
    return 0x4B400008u + static_cast<uint32_t>(asym_code_f64(h, q));
  return __float_as_uint(t);
}

// Pack 8 UNCLIPPED t-bits into one word of 4-bit two's-complement codes,
// element 0 lowest, saturating to [-8, 7] on the way (codec.py:231 clip, then
// :199-203 nibble order): code = t - bits(kMagic8) as s32, two codes per
// I2IP.S4.S32.SAT (cvt.pack.sat.s4), the earlier pairs shifted up by 8 bits
// through the third operand.  4 packs + 8 subtracts replace the per-element
// clips and the IMAD/PRMT packing.  Valid while |r| < 2^22 (magic-add range).
__device__ __forceinline__ uint32_t pack8_tbits_sat(const uint32_t *t) {
  constexpr uint32_t K = 0x4B400008u;
  uint32_t d;
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, 0;" : "=r"(d) : "r"(t[7] - K), "r"(t[6] - K));
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(t[5] - K), "r"(t[4] - K), "r"(d));
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(t[3] - K), "r"(t[2] - K), "r"(d));
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(t[1] - K), "r"(t[0] - K), "r"(d));
  return d;
}

// Four bytes (a[j] low nibble, b[j] high nibble, byte j) from s32 codes,
// saturated to [-8, 7]: one I2IP.S4.S32.SAT per byte.
__device__ __forceinline__ uint32_t pack4_pairs_sat(const uint32_t *a, const uint32_t *b) {
  uint32_t d;
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, 0;" : "=r"(d) : "r"(b[3]), "r"(a[3]));
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(b[2]), "r"(a[2]), "r"(d));
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(b[1]), "r"(a[1]), "r"(d));
  asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(b[0]), "r"(a[0]), "r"(d));
  return d;
}

// Pack 8 t-bits (elements 0..7) into one word of nibbles, element 0 lowest
// (codec.py:199-203): pairs by IMAD (hi*16 + lo keeps both nibbles in the low
// byte), bytes gathered by PRMT, the +8 offset removed by one XOR.
__device__ __forceinline__ uint32_t pack8_tbits(const uint32_t *t) {
  const uint32_t p0 = t[1] * 16u + t[0], p1 = t[3] * 16u + t[2];
  const uint32_t p2 = t[5] * 16u + t[4], p3 = t[7] * 16u + t[6];
  const uint32_t a = __byte_perm(p0, p1, 0x0040), b = __byte_perm(p2, p3, 0x0040);
  return __byte_perm(a, b, 0x5410) ^ 0x88888888u;
}

// Signed code of nibble j of a packed word.
__device__ __forceinline__ float nib_code(uint32_t w, int j) {
  uint32_t n = (w >> (4 * j)) & 0xfu;
  // (n ^ 8) - 8 sign-extends the 4-bit two's complement value.
  return __int_as_float(0x4B400000 | (n ^ 8u)) - (kMagic + 8.f);
}

// Dequantised value: code*s is exact in f32; code*s + o is one FMA rounding,
// identical to the reference's float64 sum rounded to float32 (Appendix A.8).
template <bool ASYM>
__device__ __forceinline__ float deq(float code, float s, float o) {
  return ASYM ? fmaf(code, s, o) : code * s;
}

// ---------------------------------------------------------------------------
// output stores
// ---------------------------------------------------------------------------
template <int OT>
struct Storer;

template <>
struct Storer<ADC_F32> {
  static constexpr int kBytes = 4;
  __device__ __forceinline__ static void store8(void *y, int64_t i, const float *v) {
    char *p = static_cast<char *>(y) + i * 4;
    st_stream16(p, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                              __float_as_uint(v[2]), __float_as_uint(v[3])));
    st_stream16(p + 16, make_uint4(__float_as_uint(v[4]), __float_as_uint(v[5]),
                                   __float_as_uint(v[6]), __float_as_uint(v[7])));
  }
  __device__ __forceinline__ static void store1(void *y, int64_t i, float v) {
    static_cast<float *>(y)[i] = v;
  }
};

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}

template <>
struct Storer<ADC_BF16> {
  static constexpr int kBytes = 2;
  __device__ __forceinline__ static void store8(void *y, int64_t i, const float *v) {
    st_stream16(static_cast<char *>(y) + i * 2,
                make_uint4(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]), pack_bf2(v[4], v[5]),
                           pack_bf2(v[6], v[7])));
  }
  __device__ __forceinline__ static void store1(void *y, int64_t i, float v) {
    static_cast<__nv_bfloat16 *>(y)[i] = __float2bfloat16_rn(v);
  }
};

template <>
struct Storer<ADC_F16> {
  static constexpr int kBytes = 2;
  __device__ __forceinline__ static void store8(void *y, int64_t i, const float *v) {
    st_stream16(static_cast<char *>(y) + i * 2,
                make_uint4(f32x2_to_h2(v[0], v[1]), f32x2_to_h2(v[2], v[3]),
                           f32x2_to_h2(v[4], v[5]), f32x2_to_h2(v[6], v[7])));
  }
  __device__ __forceinline__ static void store1(void *y, int64_t i, float v) {
    static_cast<__half *>(y)[i] = __float2half_rn(v);
  }
};

// gpu-scope acquire-release fetch-add (arrival counters)
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine, 1-D) pipeline primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra LAB_WAIT;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (UBLKCP), completion counted on `bar` in bytes;
// evict-first: the source is streamed once.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n\t}"
      ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Programmatic dependent launch (every kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, launch.h): wait until
// the preceding grid in the stream has completed and its memory is visible,
// and let the next grid be scheduled as soon as all of this grid's CTAs have
// started -- its launch and prologue then overlap this grid's tail.  Both
// are no-ops for a normal launch.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void raise_err(uint32_t *err, uint32_t bit) {
  if (err) atomicOr(err, bit);
}

}  // namespace adc
