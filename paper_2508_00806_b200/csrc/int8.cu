// Extension (north_star "int8/int4 ... fp32 scales"; no reference
// counterpart -- SURVEY.md 0.1, SPEC.md:240 excludes INT8): symmetric group
// int8 codes with float32 scales.  Parity is UNPINNED: the semantics are
// defined here and restated in oracle/int8_oracle.py, which the tests check
// bit-for-bit:
//   h = f16(x) (the reference's cast, codec.py:158, incl. its non-finite rule);
//   groups of g elements over the row-major flattened tensor (codec.py:183);
//   s = RN32(max|h| / 127); code = clip(rint_even(RN32(h / s')), -127, 127)
//   with s' = 1 for an all-zero group; dequantised value = RN32(code * s).
// One lane owns 8 consecutive elements (one 128-bit load of bf16/f16, two of
// f32 -> one 64-bit code store), a group of g = 8L elements sits on L lanes.
#include "common.cuh"
#include "launch.h"
#include "quant.cuh"

namespace adc {

__device__ __forceinline__ uint32_t i8_code(float h, float s) {
  float q = __fdiv_rn(h, s);  // IEEE f32 quotient (numpy float32 division)
  q = fminf(fmaxf(q, -127.f), 127.f);
  return static_cast<uint32_t>(__float2int_rn(q)) & 0xffu;  // RNE
}

// Codes clip(rint_even(RN32(h / s))) in [LO, HI] of a unit's 8 elements
// (raw f16 words w) without an IEEE division per element, two elements per
// packed f32x2 instruction: the Markstein quotient q = r0 + (h - r0*s)*inv
// (inv = rcp.approx, the residual exact by FMA) is within 1 ulp of h/s and
// RN32(h/s) within half an ulp, so the two can round to different integers
// only if q lies within 1.5 ulp (< 2^-14 for |q| < 128) of a half-integer.
// q + magic rounds to the nearest integer (ties to even); the residual
// e = q - rint(q) is exact, and e*e - T > 0 (one FFMA2 per pair; T just
// below (1/2 - 2^-14)^2, so the test errs towards redoing) marks the
// elements recomputed with the IEEE division (rare; one branch per lane).
// No clip is needed on the fast path: |q| <= 127 (resp. 8) up to an ulp, and
// the saturating pack maps rint(q) = 8 to 7 exactly as clip-then-rint does.
// Requires a finite non-zero s (non-finite groups take the exact per-element
// path).
template <int LO, int HI, int BITS>
__device__ __forceinline__ uint64_t codes8_fast(const uint32_t *w, float s, float inv) {
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  constexpr float kMg = BITS == 8 ? kMagic : kMagic8;
  constexpr float kT = (0.5f - 0x1p-14f) * (0.5f - 0x1p-14f) * (1.f - 0x1p-20f);
  const uint64_t inv2 = f2_pack(inv, inv), ns2 = f2_pack(-s, -s), mg2 = f2_pack(kMg, kMg);
  const uint64_t nt2 = f2_pack(-kT, -kT);
  uint32_t t[8], signs = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t h2 = f2_pack(lo_f(w[i]), hi_f(w[i]));
    const uint64_t r0 = f2_mul(h2, inv2);
    const uint64_t r1 = f2_fma(f2_fma(r0, ns2, h2), inv2, r0);
    const uint64_t tv2 = f2_add(r1, mg2);
    const uint64_t e2 = f2_sub(r1, f2_sub(tv2, mg2));
    float dl, dh, tl, th;
    f2_unpack(f2_fma(e2, e2, nt2), dl, dh);
    signs = __funnelshift_l(__float_as_uint(dl), signs, 1);
    signs = __funnelshift_l(__float_as_uint(dh), signs, 1);
    f2_unpack(tv2, tl, th);
    t[2 * i] = __float_as_uint(tl);
    t[2 * i + 1] = __float_as_uint(th);
  }
  const uint32_t fix = ~__brev(signs) >> 24;  // element j at bit j: e*e >= T
  uint64_t out;
  if (BITS == 8) {
    constexpr uint32_t K = 0x4B400000u;  // bits of kMagic: t - K = rint(q) as s32
    uint32_t lo, hi, d;
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(d) : "r"(t[3] - K), "r"(t[2] - K));
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(t[1] - K), "r"(t[0] - K), "r"(d));
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(d) : "r"(t[7] - K), "r"(t[6] - K));
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(hi) : "r"(t[5] - K), "r"(t[4] - K), "r"(d));
    out = static_cast<uint64_t>(lo) | (static_cast<uint64_t>(hi) << 32);
  } else {
    out = pack8_tbits_sat(t);
  }
  if (fix) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (fix & (1u << j)) {
        const float h = (j & 1) ? hi_f(w[j >> 1]) : lo_f(w[j >> 1]);
        const float qe = fminf(fmaxf(__fdiv_rn(h, s), static_cast<float>(LO)), static_cast<float>(HI));
        const uint64_t code = static_cast<uint32_t>(__float2int_rn(qe)) & kMask;
        out = (out & ~(static_cast<uint64_t>(kMask) << (BITS * j))) | (code << (BITS * j));
      }
    }
  }
  return out;
}

// RN32(top / 127) for an f16 top: Markstein's correction with the correctly
// rounded reciprocal -- checked against IEEE division for every finite f16
// value (tests/test_int8_extension.py::test_int8_scale_division_exhaustive)
__device__ __forceinline__ float div127(float top) {
  constexpr float y = 1.0f / 127.0f;
  const float q0 = __fmul_rn(top, y);
  return __fmaf_rn(__fmaf_rn(-q0, 127.0f, top), y, q0);
}

// U units (8 elements each) per lane in flight: their loads are issued
// before any is processed
template <int DT, int L, int U>
__global__ void __launch_bounds__(kThreads)
    int8_quant(const void *__restrict__ x, int64_t n_units, int64_t n_units_pad,
               uint2 *__restrict__ codes, float *__restrict__ scales, uint32_t *__restrict__ err) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads * U;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads * U; base < n_units_pad; base += step) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      v[k] = u < n_units ? Loader<DT>::template load8<false>(x, u * 8) : make_uint4(0, 0, 0, 0);  // f16 words
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;  // groups never straddle warps
      const bool act = u < n_units;
      const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
      uint32_t m = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) m = __vmaxu2(m, w[i] & 0x7fff7fffu);
      m = warp_max_u2<L>(m);
      const uint32_t top = max(m & 0xffffu, m >> 16);
      const bool fin = top < 0x7c00u;  // finite scale: the division-free codes
      const float s = fin ? div127(h2f(top)) : __fdiv_rn(h2f(top), 127.f);
      const float sd = s == 0.f ? 1.f : s;
      if (act) {
        if (fin) {
          const uint64_t cc = codes8_fast<-127, 127, 8>(w, sd, rcp_approx(sd));
          codes[u] = make_uint2(static_cast<uint32_t>(cc), static_cast<uint32_t>(cc >> 32));
        } else {
          uint32_t lo = 0, hi = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t pair = i8_code(lo_f(w[j]), sd) | (i8_code(hi_f(w[j]), sd) << 8);
            if (j < 2)
              lo |= pair << (16 * j);
            else
              hi |= pair << (16 * (j - 2));
          }
          codes[u] = make_uint2(lo, hi);
        }
      }
      if ((threadIdx.x & (L - 1)) == 0 && u < n_units_pad) {
        scales[u / L] = s;
        if (top >= 0x7c00u) raise_err(err, ADC_ERR_NONFINITE);
      }
    }
  }
}

// Any shape / group size: one warp per group, element-wise.
template <int DT>
__global__ void __launch_bounds__(kThreads)
    int8_quant_generic(const void *__restrict__ x, int64_t n, int64_t g, int8_t *__restrict__ codes,
                       float *__restrict__ scales, uint32_t *__restrict__ err) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t n_groups = (n + g - 1) / g;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + threadIdx.x / 32; j < n_groups;
       j += warps) {
    const int64_t e0 = j * g, cnt = min(g, n - e0);
    uint32_t top = 0;
    for (int64_t i = lane; i < cnt; i += 32) top = max(top, Loader<DT>::load1(x, e0 + i) & 0x7fffu);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
    const float s = __fdiv_rn(h2f(top), 127.f);
    const float sd = s == 0.f ? 1.f : s;
    for (int64_t i = lane; i < cnt; i += 32)
      codes[e0 + i] = static_cast<int8_t>(i8_code(h2f(Loader<DT>::load1(x, e0 + i)), sd));
    if (lane == 0) {
      scales[j] = s;
      if (top >= 0x7c00u) raise_err(err, ADC_ERR_NONFINITE);
    }
  }
}

template <int OT>
__global__ void __launch_bounds__(kThreads)
    int8_dequant(const int8_t *__restrict__ codes, const float *__restrict__ scales, int64_t n,
                 int64_t g, void *__restrict__ y) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads;
  const int64_t n8 = n / 8;
  for (int64_t u = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; u < n8; u += step) {
    const uint2 c = __ldcs(reinterpret_cast<const uint2 *>(codes) + u);
    const uint32_t cw[2] = {c.x, c.y};
    float v[8];
    if (g % 8 == 0) {
      const float s = __ldg(scales + (u * 8) / g);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[j] = static_cast<float>(static_cast<int8_t>((cw[j >> 2] >> (8 * (j & 3))) & 0xffu)) * s;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[j] = static_cast<float>(static_cast<int8_t>((cw[j >> 2] >> (8 * (j & 3))) & 0xffu)) *
               __ldg(scales + (u * 8 + j) / g);
    }
    Storer<OT>::store8(y, u * 8, v);
  }
  for (int64_t e = n8 * 8 + static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; e < n; e += step)
    Storer<OT>::store1(y, e, static_cast<float>(codes[e]) * __ldg(scales + e / g));
}

// g = 8 * 2^shift, n % 8 == 0: the group of unit u is u >> shift (no
// division), U units per lane with their code and scale loads in flight
template <int OT, int U>
__global__ void __launch_bounds__(kThreads)
    int8_dequant_fast(const uint2 *__restrict__ codes, const float *__restrict__ scales, int64_t n8, int shift,
                      void *__restrict__ y) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads * U;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads * U; base < n8; base += step) {
    uint2 c[U];
    float s[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      c[k] = u < n8 ? __ldcs(codes + u) : make_uint2(0, 0);
      s[k] = u < n8 ? __ldg(scales + (u >> shift)) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      if (u >= n8) continue;
      const uint32_t cw[2] = {c[k].x, c[k].y};
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[j] = static_cast<float>(static_cast<int8_t>((cw[j >> 2] >> (8 * (j & 3))) & 0xffu)) * s[k];
      Storer<OT>::store8(y, u * 8, v);
    }
  }
}

constexpr int kUI8 = 4;  // units per lane in flight (int8 / int4-f32 fast kernels)

static inline int pow2_shift(int64_t v) {  // log2(v) if v is a power of two, else -1
  if (v < 1 || (v & (v - 1))) return -1;
  int sh = 0;
  while ((int64_t{1} << sh) < v) ++sh;
  return sh;
}

static inline int grid_i8(const Ctx &c, int64_t items) {
  int64_t need = (items + kThreads - 1) / kThreads;
  const int64_t cap = static_cast<int64_t>(c.num_sms) * 8;
  return static_cast<int>(need < 1 ? 1 : (need < cap ? need : cap));
}

int launch_int8_compress(const Ctx &c, const void *x, int dt, int64_t n, int64_t g, int8_t *codes,
                         float *scales, uint32_t *err) {
  const int64_t L = g / 8;
  const bool fast = g % 8 == 0 && L >= 1 && L <= 32 && (L & (L - 1)) == 0 && n % 8 == 0 &&
                    reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(codes) % 8 == 0;
#define ADC_I8_DT(DTV, BODY)                                     \
  switch (DTV) {                                                 \
    case ADC_F32: { constexpr int DT = ADC_F32; BODY; break; }   \
    case ADC_BF16: { constexpr int DT = ADC_BF16; BODY; break; } \
    case ADC_F16: { constexpr int DT = ADC_F16; BODY; break; }   \
    default: return -1;                                          \
  }
  if (fast) {
    const int64_t n_units = n / 8, n_units_pad = (n_units + L - 1) / L * L;
    const int grid = grid_i8(c, (n_units_pad + kUI8 - 1) / kUI8);
    uint2 *c2 = reinterpret_cast<uint2 *>(codes);
#define ADC_I8_L(LV) \
  case LV: ADC_I8_DT(dt, launch_k(int8_quant<DT, LV, kUI8>, grid, kThreads, 0, c.stream, x, n_units, n_units_pad, c2, scales, err)); break;
    switch (L) {
      ADC_I8_L(1) ADC_I8_L(2) ADC_I8_L(4) ADC_I8_L(8) ADC_I8_L(16) ADC_I8_L(32)
      default: return -1;
    }
#undef ADC_I8_L
  } else {
    const int grid = grid_i8(c, ((n + g - 1) / g) * 32);
    ADC_I8_DT(dt, launch_k(int8_quant_generic<DT>, grid, kThreads, 0, c.stream, x, n, g, codes, scales, err));
  }
#undef ADC_I8_DT
  note_launches(1);
  return 0;
}

int launch_int8_decompress(const Ctx &c, const int8_t *codes, const float *scales, int64_t n, int64_t g,
                           void *y, int ot) {
  if (reinterpret_cast<uintptr_t>(codes) % 8 || reinterpret_cast<uintptr_t>(y) % 16) return -1;
  const int sh = g % 8 == 0 ? pow2_shift(g / 8) : -1;
  if (sh >= 0 && n % 8 == 0) {
    const int64_t n8 = n / 8;
    const int gf = grid_i8(c, (n8 + kUI8 - 1) / kUI8);
    const uint2 *c2 = reinterpret_cast<const uint2 *>(codes);
    switch (ot) {
      case ADC_F32: launch_k(int8_dequant_fast<ADC_F32, kUI8>, gf, kThreads, 0, c.stream, c2, scales, n8, sh, y); break;
      case ADC_BF16: launch_k(int8_dequant_fast<ADC_BF16, kUI8>, gf, kThreads, 0, c.stream, c2, scales, n8, sh, y); break;
      case ADC_F16: launch_k(int8_dequant_fast<ADC_F16, kUI8>, gf, kThreads, 0, c.stream, c2, scales, n8, sh, y); break;
      default: return -1;
    }
    note_launches(1);
    return 0;
  }
  const int grid = grid_i8(c, n / 8 + 1);
  switch (ot) {
    case ADC_F32: launch_k(int8_dequant<ADC_F32>, grid, kThreads, 0, c.stream, codes, scales, n, g, y); break;
    case ADC_BF16: launch_k(int8_dequant<ADC_BF16>, grid, kThreads, 0, c.stream, codes, scales, n, g, y); break;
    case ADC_F16: launch_k(int8_dequant<ADC_F16>, grid, kThreads, 0, c.stream, codes, scales, n, g, y); break;
    default: return -1;
  }
  note_launches(1);
  return 0;
}

// ---------------------------------------------------------------------------
// Extension: the int4 symmetric group codec with FLOAT32 scales (north_star
// "fp32-scale storage option"; the reference rounds every scale to float16,
// codec.py:192-196).  Parity UNPINNED, restated in oracle/int8_oracle.py:
//   h = f16(x); s = RN32(max|h| / 8) (exact: a power-of-two divisor);
//   code = clip(rint_even(RN32(h / s')), -8, 7), s' = 1 for an all-zero
//   group; nibbles packed as the reference's (element 2i in the low nibble,
//   codec.py:199-203); dequantised value = RN32(code * s).
// Same lane layout as the int8 kernels: 8 elements per lane -> one 32-bit
// code word, a group of g = 8L elements on L lanes.
__device__ __forceinline__ uint32_t i4_code(float h, float s) {
  float q = __fdiv_rn(h, s);
  q = fminf(fmaxf(q, -8.f), 7.f);
  return static_cast<uint32_t>(__float2int_rn(q)) & 0xfu;
}

template <int DT, int L, int U>
__global__ void __launch_bounds__(kThreads)
    int4f32_quant(const void *__restrict__ x, int64_t n_units, int64_t n_units_pad, uint32_t *__restrict__ codes,
                  float *__restrict__ scales, uint32_t *__restrict__ err) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads * U;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads * U; base < n_units_pad; base += step) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      v[k] = u < n_units ? Loader<DT>::template load8<false>(x, u * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;  // groups never straddle warps
      const bool act = u < n_units;
      const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
      uint32_t m = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) m = __vmaxu2(m, w[i] & 0x7fff7fffu);
      m = warp_max_u2<L>(m);
      const uint32_t top = max(m & 0xffffu, m >> 16);
      const float s = h2f(top) * 0.125f;
      const float sd = s == 0.f ? 1.f : s;
      const bool fin = top < 0x7c00u;  // finite scale: the division-free codes
      if (act) {
        uint32_t cw = 0;
        if (fin) {
          cw = static_cast<uint32_t>(codes8_fast<-8, 7, 4>(w, sd, rcp_approx(sd)));
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            cw |= (i4_code(lo_f(w[j]), sd) | (i4_code(hi_f(w[j]), sd) << 4)) << (8 * j);
        }
        codes[u] = cw;
      }
      if ((threadIdx.x & (L - 1)) == 0 && u < n_units_pad) {
        scales[u / L] = s;
        if (top >= 0x7c00u) raise_err(err, ADC_ERR_NONFINITE);
      }
    }
  }
}

// Any shape / group size: one warp per group, element-wise (nibble bytes
// assembled from element pairs; a pair may straddle two groups).
template <int DT>
__global__ void __launch_bounds__(kThreads)
    int4f32_scales_generic(const void *__restrict__ x, int64_t n, int64_t g, float *__restrict__ scales,
                           uint32_t *__restrict__ err) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t n_groups = (n + g - 1) / g;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + threadIdx.x / 32; j < n_groups;
       j += warps) {
    const int64_t e0 = j * g, cnt = min(g, n - e0);
    uint32_t top = 0;
    for (int64_t i = lane; i < cnt; i += 32) top = max(top, Loader<DT>::load1(x, e0 + i) & 0x7fffu);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
    if (lane == 0) {
      scales[j] = h2f(top) * 0.125f;
      if (top >= 0x7c00u) raise_err(err, ADC_ERR_NONFINITE);
    }
  }
}
template <int DT>
__global__ void __launch_bounds__(kThreads)
    int4f32_codes_generic(const void *__restrict__ x, int64_t n, int64_t g, const float *__restrict__ scales,
                          uint8_t *__restrict__ codes) {
  pdl_entry();
  const int64_t nb = (n + 1) / 2;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * kThreads) {
    uint32_t byte = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int64_t e = 2 * b + k;
      if (e < n) {
        const float s = scales[e / g];
        byte |= i4_code(h2f(Loader<DT>::load1(x, e)), s == 0.f ? 1.f : s) << (4 * k);
      }
    }
    codes[b] = static_cast<uint8_t>(byte);
  }
}

template <int OT, int U>
__global__ void __launch_bounds__(kThreads)
    int4f32_dequant_fast(const uint32_t *__restrict__ codes, const float *__restrict__ scales, int64_t n8,
                         int shift, void *__restrict__ y) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads * U;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads * U; base < n8; base += step) {
    uint32_t c[U];
    float s[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      c[k] = u < n8 ? __ldcs(codes + u) : 0u;
      s[k] = u < n8 ? __ldg(scales + (u >> shift)) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      if (u >= n8) continue;
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = nib_code(c[k], j) * s[k];
      Storer<OT>::store8(y, u * 8, v);
    }
  }
}

template <int OT>
__global__ void __launch_bounds__(kThreads)
    int4f32_dequant(const uint8_t *__restrict__ codes, const float *__restrict__ scales, int64_t n, int64_t g,
                    void *__restrict__ y) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads;
  const int64_t n8 = n / 8;
  for (int64_t u = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; u < n8; u += step) {
    const uint32_t cw = __ldcs(reinterpret_cast<const uint32_t *>(codes) + u);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float s = g % 8 == 0 ? __ldg(scales + (u * 8) / g) : __ldg(scales + (u * 8 + j) / g);
      v[j] = nib_code(cw, j) * s;
    }
    Storer<OT>::store8(y, u * 8, v);
  }
  for (int64_t e = n8 * 8 + static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; e < n; e += step) {
    const uint32_t byte = codes[e / 2];
    Storer<OT>::store1(y, e, nib_code(byte, static_cast<int>(e & 1)) * __ldg(scales + e / g));
  }
}

int launch_int4f32_compress(const Ctx &c, const void *x, int dt, int64_t n, int64_t g, uint8_t *codes,
                            float *scales, uint32_t *err) {
  const int64_t L = g / 8;
  const bool fast = g % 8 == 0 && L >= 1 && L <= 32 && (L & (L - 1)) == 0 && n % 8 == 0 &&
                    reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(codes) % 4 == 0;
#define ADC_I4_DT(DTV, BODY)                                     \
  switch (DTV) {                                                 \
    case ADC_F32: { constexpr int DT = ADC_F32; BODY; break; }   \
    case ADC_BF16: { constexpr int DT = ADC_BF16; BODY; break; } \
    case ADC_F16: { constexpr int DT = ADC_F16; BODY; break; }   \
    default: return -1;                                          \
  }
  if (fast) {
    const int64_t n_units = n / 8, n_units_pad = (n_units + L - 1) / L * L;
    const int grid = grid_i8(c, (n_units_pad + kUI8 - 1) / kUI8);
    uint32_t *c4 = reinterpret_cast<uint32_t *>(codes);
#define ADC_I4_L(LV) \
  case LV: ADC_I4_DT(dt, launch_k(int4f32_quant<DT, LV, kUI8>, grid, kThreads, 0, c.stream, x, n_units, n_units_pad, c4, scales, err)); break;
    switch (L) {
      ADC_I4_L(1) ADC_I4_L(2) ADC_I4_L(4) ADC_I4_L(8) ADC_I4_L(16) ADC_I4_L(32)
      default: return -1;
    }
#undef ADC_I4_L
    note_launches(1);
  } else {
    ADC_I4_DT(dt, launch_k(int4f32_scales_generic<DT>, grid_i8(c, ((n + g - 1) / g) * 32), kThreads, 0, c.stream,
                           x, n, g, scales, err));
    ADC_I4_DT(dt, launch_k(int4f32_codes_generic<DT>, grid_i8(c, (n + 1) / 2), kThreads, 0, c.stream, x, n, g,
                           scales, codes));
    note_launches(2);
  }
#undef ADC_I4_DT
  return 0;
}

int launch_int4f32_decompress(const Ctx &c, const uint8_t *codes, const float *scales, int64_t n, int64_t g,
                              void *y, int ot) {
  if (reinterpret_cast<uintptr_t>(codes) % 4 || reinterpret_cast<uintptr_t>(y) % 16) return -1;
  const int sh = g % 8 == 0 ? pow2_shift(g / 8) : -1;
  if (sh >= 0 && n % 8 == 0) {
    const int64_t n8 = n / 8;
    const int gf = grid_i8(c, (n8 + kUI8 - 1) / kUI8);
    const uint32_t *c4 = reinterpret_cast<const uint32_t *>(codes);
    switch (ot) {
      case ADC_F32: launch_k(int4f32_dequant_fast<ADC_F32, kUI8>, gf, kThreads, 0, c.stream, c4, scales, n8, sh, y); break;
      case ADC_BF16: launch_k(int4f32_dequant_fast<ADC_BF16, kUI8>, gf, kThreads, 0, c.stream, c4, scales, n8, sh, y); break;
      case ADC_F16: launch_k(int4f32_dequant_fast<ADC_F16, kUI8>, gf, kThreads, 0, c.stream, c4, scales, n8, sh, y); break;
      default: return -1;
    }
    note_launches(1);
    return 0;
  }
  const int grid = grid_i8(c, n / 8 + 1);
  switch (ot) {
    case ADC_F32: launch_k(int4f32_dequant<ADC_F32>, grid, kThreads, 0, c.stream, codes, scales, n, g, y); break;
    case ADC_BF16: launch_k(int4f32_dequant<ADC_BF16>, grid, kThreads, 0, c.stream, codes, scales, n, g, y); break;
    case ADC_F16: launch_k(int4f32_dequant<ADC_F16>, grid, kThreads, 0, c.stream, codes, scales, n, g, y); break;
    default: return -1;
  }
  note_launches(1);
  return 0;
}

}  // namespace adc
