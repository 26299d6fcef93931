// K5: dropout-mask bit packing (scheme_for(DROPOUT_MASK), codec.py:80-81).
//
// Reference: pack_bitmask (codec.py:344-369) -- bytes must be 0/1
// (NonBinaryMaskError otherwise), bit (i mod 8) of byte i/8 = m[i]
// (np.packbits bitorder="little"), zero padding; unpack_bitmask (:372-378).
// One thread packs 64 elements into one 64-bit word.
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace adc {

// 4 bytes in {0,1} (u32) -> 4 bits; multiplier places byte j's bit 0 at bit 24+j
__device__ __forceinline__ uint32_t gather4(uint32_t w) { return ((w * 0x01020408u) >> 24) & 0xfu; }
// 4 bits -> 4 bytes in {0,1}
__device__ __forceinline__ uint32_t spread4(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

template <int DT>
struct MaskIn;

template <>
struct MaskIn<ADC_U8> {
  // 8 elements -> 8 bits; bad if any byte not in {0,1}
  __device__ __forceinline__ static uint32_t bits8(const void *m, int64_t i, bool &bad) {
    const uint2 v = *reinterpret_cast<const uint2 *>(static_cast<const uint8_t *>(m) + i);
    bad |= ((v.x | v.y) & 0xfefefefeu) != 0;
    return gather4(v.x) | (gather4(v.y) << 4);
  }
  __device__ __forceinline__ static uint32_t bit1(const void *m, int64_t i, bool &bad) {
    const uint32_t b = static_cast<const uint8_t *>(m)[i];
    bad |= b > 1;
    return b & 1u;
  }
};

template <typename T>
__device__ __forceinline__ uint32_t fbit(T v, bool &bad) {
  const float f = static_cast<float>(v);
  bad |= !(f == 0.f || f == 1.f);
  return f == 1.f;
}

template <>
struct MaskIn<ADC_F32> {
  __device__ __forceinline__ static uint32_t bits8(const void *m, int64_t i, bool &bad) {
    const float4 *p = reinterpret_cast<const float4 *>(static_cast<const float *>(m) + i);
    const float4 a = p[0], b = p[1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r |= fbit(v[j], bad) << j;
    return r;
  }
  __device__ __forceinline__ static uint32_t bit1(const void *m, int64_t i, bool &bad) {
    return fbit(static_cast<const float *>(m)[i], bad);
  }
};

template <>
struct MaskIn<ADC_BF16> {
  __device__ __forceinline__ static uint32_t bits8(const void *m, int64_t i, bool &bad) {
    const uint4 v = *reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(m) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float f = __uint_as_float(((w[j >> 1] >> ((j & 1) * 16)) & 0xffffu) << 16);
      r |= fbit(f, bad) << j;
    }
    return r;
  }
  __device__ __forceinline__ static uint32_t bit1(const void *m, int64_t i, bool &bad) {
    const uint32_t u = static_cast<const uint16_t *>(m)[i];
    return fbit(__uint_as_float(u << 16), bad);
  }
};

template <>
struct MaskIn<ADC_F16> {
  __device__ __forceinline__ static uint32_t bits8(const void *m, int64_t i, bool &bad) {
    const uint4 v = *reinterpret_cast<const uint4 *>(static_cast<const uint16_t *>(m) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r |= fbit(h2f((w[j >> 1] >> ((j & 1) * 16)) & 0xffffu), bad) << j;
    return r;
  }
  __device__ __forceinline__ static uint32_t bit1(const void *m, int64_t i, bool &bad) {
    return fbit(h2f(static_cast<const uint16_t *>(m)[i]), bad);
  }
};

// FAST: n % 8 == 0 and vector-aligned input; else byte-by-byte.
template <int DT, bool FAST>
__global__ void __launch_bounds__(kThreads)
    mask_pack(const void *__restrict__ m, int64_t n, uint8_t *__restrict__ bits,
              uint32_t *__restrict__ err) {
  pdl_entry();
  const int64_t nbytes = (n + 7) / 8;
  bool bad = false;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; b < nbytes;
       b += static_cast<int64_t>(gridDim.x) * kThreads) {
    uint32_t v = 0;
    if (FAST) {
      v = MaskIn<DT>::bits8(m, b * 8, bad);
    } else {
      for (int j = 0; j < 8 && b * 8 + j < n; ++j) v |= MaskIn<DT>::bit1(m, b * 8 + j, bad) << j;
    }
    bits[b] = static_cast<uint8_t>(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_err(err, ADC_ERR_NONBINARY);
}

// One thread expands one packed byte into 8 output bytes (a u64 store).
template <bool FAST>
__global__ void __launch_bounds__(kThreads)
    mask_unpack(const uint8_t *__restrict__ bits, int64_t n, uint8_t *__restrict__ out) {
  pdl_entry();
  const int64_t nbytes = (n + 7) / 8;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; b < nbytes;
       b += static_cast<int64_t>(gridDim.x) * kThreads) {
    const uint32_t v = bits[b];
    if (FAST) {
      *reinterpret_cast<uint2 *>(out + b * 8) = make_uint2(spread4(v & 0xfu), spread4(v >> 4));
    } else {
      for (int j = 0; j < 8 && b * 8 + j < n; ++j) out[b * 8 + j] = (v >> j) & 1u;
    }
  }
}

// Wide variants for byte masks (bool tensors, the training case): a thread
// packs 32 elements (two 128-bit loads -> one 32-bit store, two units in
// flight); the inverse expands 16-bit pieces into 128-bit stores.
__global__ void __launch_bounds__(kThreads)
    mask_pack_u8x32(const uint4 *__restrict__ m, int64_t units, uint32_t *__restrict__ bits,
                    uint32_t *__restrict__ err) {
  pdl_entry();
  bool bad = false;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
  for (int64_t u = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; u < units; u += 2 * stride) {
    uint4 v[2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t uq = u + q * stride;
      v[q][0] = uq < units ? __ldcs(m + 2 * uq) : make_uint4(0, 0, 0, 0);
      v[q][1] = uq < units ? __ldcs(m + 2 * uq + 1) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t uq = u + q * stride;
      if (uq >= units) continue;
      const uint32_t w[8] = {v[q][0].x, v[q][0].y, v[q][0].z, v[q][0].w,
                             v[q][1].x, v[q][1].y, v[q][1].z, v[q][1].w};
      uint32_t r = 0, any = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        any |= w[j];
        r |= gather4(w[j]) << (4 * j);
      }
      bad |= (any & 0xfefefefeu) != 0;
      __stcs(bits + uq, r);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) raise_err(err, ADC_ERR_NONBINARY);
}

__global__ void __launch_bounds__(kThreads)
    mask_unpack_u8x32(const uint32_t *__restrict__ bits, int64_t units, uint4 *__restrict__ out) {
  // units of 32 elements; a warp expands 32 units = 1024 bytes per round:
  // lane l takes the 16-bit halves l and 32 + l of the warp's 32 mask words,
  // so each 128-bit store instruction covers 512 contiguous output bytes
  pdl_entry();
  const uint16_t *b16 = reinterpret_cast<const uint16_t *>(bits);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t n_warps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  const int64_t halves = 2 * units;  // 16-element pieces
  for (int64_t w0 = warp * 64; w0 < halves; w0 += n_warps * 64) {
    const int64_t pa = w0 + lane, pb = w0 + 32 + lane;
    const uint32_t a = pa < halves ? __ldcs(b16 + pa) : 0u, b = pb < halves ? __ldcs(b16 + pb) : 0u;
    if (pa < halves)
      out[pa] = make_uint4(spread4(a & 0xfu), spread4((a >> 4) & 0xfu), spread4((a >> 8) & 0xfu),
                           spread4(a >> 12));
    if (pb < halves)
      out[pb] = make_uint4(spread4(b & 0xfu), spread4((b >> 4) & 0xfu), spread4((b >> 8) & 0xfu),
                           spread4(b >> 12));
  }
}

static bool use_wide_unpack() {
  const char *e = getenv("ADC_MASK_WIDE_UNPACK");
  return !(e && e[0] == '0');
}

static inline int grid_of(const Ctx &c, int64_t items) {
  int64_t need = (items + kThreads - 1) / kThreads;
  int64_t cap = static_cast<int64_t>(c.num_sms) * 16;
  return static_cast<int>(need < 1 ? 1 : (need < cap ? need : cap));
}

int launch_mask_pack(const Ctx &c, const void *m, int dt, int64_t n, uint8_t *bits,
                     uint32_t *err) {
  const int elt = dt == ADC_F32 ? 4 : (dt == ADC_U8 ? 1 : 2);
  const bool fast = n % 8 == 0 && reinterpret_cast<uintptr_t>(m) % (8 * elt < 16 ? 8 * elt : 16) == 0;
  if (dt == ADC_U8 && n % 32 == 0 && reinterpret_cast<uintptr_t>(m) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(bits) % 4 == 0) {
    const int64_t units = n / 32;
    const int g = grid_of(c, (units + 1) / 2);
    launch_k(mask_pack_u8x32, g, kThreads, 0, c.stream, reinterpret_cast<const uint4 *>(m), units,
             reinterpret_cast<uint32_t *>(bits), err);
    note_launches(1);
    return 0;
  }
  const int grid = grid_of(c, (n + 7) / 8);
#define ADC_MASK_CASE(DT)                                                                    \
  case DT:                                                                                   \
    if (fast)                                                                                \
      launch_k(mask_pack<DT, true>, grid, kThreads, 0, c.stream, m, n, bits, err), note_launches(1);                 \
    else                                                                                     \
      launch_k(mask_pack<DT, false>, grid, kThreads, 0, c.stream, m, n, bits, err), note_launches(1);                \
    break;
  switch (dt) {
    ADC_MASK_CASE(ADC_U8)
    ADC_MASK_CASE(ADC_F32)
    ADC_MASK_CASE(ADC_BF16)
    ADC_MASK_CASE(ADC_F16)
    default: return -1;
  }
#undef ADC_MASK_CASE
  return 0;
}

int launch_mask_unpack(const Ctx &c, const uint8_t *bits, int64_t n, uint8_t *out) {
  // 128-bit stores covering 512 contiguous bytes per warp instruction:
  // 27.9 us vs 32.7 us for the byte-per-thread kernel at 134 MB
  if (use_wide_unpack() && n % 32 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(bits) % 4 == 0) {
    const int64_t units = n / 32;
    const int g = grid_of(c, units);
    launch_k(mask_unpack_u8x32, g, kThreads, 0, c.stream, reinterpret_cast<const uint32_t *>(bits), units,
             reinterpret_cast<uint4 *>(out));
    note_launches(1);
    return 0;
  }
  const bool fast = n % 8 == 0 && reinterpret_cast<uintptr_t>(out) % 8 == 0;
  const int grid = grid_of(c, (n + 7) / 8);
  if (fast)
    launch_k(mask_unpack<true>, grid, kThreads, 0, c.stream, bits, n, out), note_launches(1);
  else
    launch_k(mask_unpack<false>, grid, kThreads, 0, c.stream, bits, n, out), note_launches(1);
  return 0;
}

}  // namespace adc
