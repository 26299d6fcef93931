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

template <int DT, int L>
__global__ void __launch_bounds__(kThreads)
    int8_quant(const void *__restrict__ x, int64_t n_units, int64_t n_units_pad,
               uint2 *__restrict__ codes, float *__restrict__ scales, uint32_t *__restrict__ err) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads; base < n_units_pad; base += step) {
    const int64_t u = base + threadIdx.x;  // groups never straddle warps: uniform trip count
    const bool act = u < n_units;
    const uint4 v = act ? Loader<DT>::template load8<false>(x, u * 8) : make_uint4(0, 0, 0, 0);  // f16 words
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) m = __vmaxu2(m, w[i] & 0x7fff7fffu);
    m = warp_max_u2<L>(m);
    const uint32_t top = max(m & 0xffffu, m >> 16);
    const float s = __fdiv_rn(h2f(top), 127.f);
    const float sd = s == 0.f ? 1.f : s;
    if (act) {
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t c0 = i8_code(lo_f(w[j]), sd), c1 = i8_code(hi_f(w[j]), sd);
        const uint32_t pair = c0 | (c1 << 8);
        if (j < 2)
          lo |= pair << (16 * j);
        else
          hi |= pair << (16 * (j - 2));
      }
      codes[u] = make_uint2(lo, hi);
    }
    if ((threadIdx.x & (L - 1)) == 0 && u < n_units_pad) {
      scales[u / L] = s;
      if (top >= 0x7c00u) raise_err(err, ADC_ERR_NONFINITE);
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
    const int grid = grid_i8(c, n_units_pad);
    uint2 *c2 = reinterpret_cast<uint2 *>(codes);
#define ADC_I8_L(LV) \
  case LV: ADC_I8_DT(dt, launch_k(int8_quant<DT, LV>, grid, kThreads, 0, c.stream, x, n_units, n_units_pad, c2, scales, err)); break;
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

template <int DT, int L>
__global__ void __launch_bounds__(kThreads)
    int4f32_quant(const void *__restrict__ x, int64_t n_units, int64_t n_units_pad, uint32_t *__restrict__ codes,
                  float *__restrict__ scales, uint32_t *__restrict__ err) {
  pdl_entry();
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads; base < n_units_pad; base += step) {
    const int64_t u = base + threadIdx.x;  // groups never straddle warps: uniform trip count
    const bool act = u < n_units;
    const uint4 v = act ? Loader<DT>::template load8<false>(x, u * 8) : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) m = __vmaxu2(m, w[i] & 0x7fff7fffu);
    m = warp_max_u2<L>(m);
    const uint32_t top = max(m & 0xffffu, m >> 16);
    const float s = h2f(top) * 0.125f;
    const float sd = s == 0.f ? 1.f : s;
    if (act) {
      uint32_t cw = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        cw |= (i4_code(lo_f(w[j]), sd) | (i4_code(hi_f(w[j]), sd) << 4)) << (8 * j);
      codes[u] = cw;
    }
    if ((threadIdx.x & (L - 1)) == 0 && u < n_units_pad) {
      scales[u / L] = s;
      if (top >= 0x7c00u) raise_err(err, ADC_ERR_NONFINITE);
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
    const int grid = grid_i8(c, n_units_pad);
    uint32_t *c4 = reinterpret_cast<uint32_t *>(codes);
#define ADC_I4_L(LV) \
  case LV: ADC_I4_DT(dt, launch_k(int4f32_quant<DT, LV>, grid, kThreads, 0, c.stream, x, n_units, n_units_pad, c4, scales, err)); break;
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
