// K1/K2/K4-quantise on a TMA-fed pipeline: the streaming compress kernel.
//
// Same semantics as group_quant_fast (group.cu; reference _quantize,
// codec.py:216-242, and the outlier zeroing of compress_outlier_separated,
// codec.py:328-340), different memory engine:
//   * one producer lane per CTA issues 1-D bulk copies (cp.async.bulk,
//     the TMA engine) of 16 KB input tiles into a 4-stage shared-memory ring,
//     completion tracked by mbarrier transaction counts;
//   * 16 consumer warps quantise a tile from shared memory (conflict-free
//     128-bit LDS, 8 elements per lane, a group of g = 8L elements on L lanes)
//     and store codes / scales straight to global;
//   * 2 CTAs per SM, persistent over tiles, so up to 128 KB per SM is in
//     flight while the math runs -- the register-prefetch version stalled on
//     load latency between its serial batches.
#include "common.cuh"
#include "launch.h"

namespace adc {

constexpr int kTileBytes = 16384;
constexpr int kStages = 4;
constexpr int kConsumerWarps = 16;
constexpr int kStreamThreads = (kConsumerWarps + 1) * 32;
constexpr int kStreamSmem = kStages * kTileBytes;

template <int DT>
__device__ __forceinline__ uint4 smem_load8(const unsigned char *tile, int j);

template <>
__device__ __forceinline__ uint4 smem_load8<ADC_F16>(const unsigned char *tile, int j) {
  return *reinterpret_cast<const uint4 *>(tile + 16 * j);
}
template <>
__device__ __forceinline__ uint4 smem_load8<ADC_BF16>(const unsigned char *tile, int j) {
  const uint4 v = *reinterpret_cast<const uint4 *>(tile + 16 * j);
  return make_uint4(bf2_to_h2(v.x), bf2_to_h2(v.y), bf2_to_h2(v.z), bf2_to_h2(v.w));
}
template <>
__device__ __forceinline__ uint4 smem_load8<ADC_F32>(const unsigned char *tile, int j) {
  const uint4 a = *reinterpret_cast<const uint4 *>(tile + 32 * j);
  const uint4 b = *reinterpret_cast<const uint4 *>(tile + 32 * j + 16);
  return make_uint4(f32x2_to_h2(__uint_as_float(a.x), __uint_as_float(a.y)),
                    f32x2_to_h2(__uint_as_float(a.z), __uint_as_float(a.w)),
                    f32x2_to_h2(__uint_as_float(b.x), __uint_as_float(b.y)),
                    f32x2_to_h2(__uint_as_float(b.z), __uint_as_float(b.w)));
}

__device__ __forceinline__ uint32_t fdiv_u32(uint32_t n, const FastDiv &f) {
  return static_cast<uint32_t>((static_cast<uint64_t>(n) * f.m) >> f.p);
}

// rare path of the outlier zeroing (values are gathered separately)
__device__ __forceinline__ void stream_zero_hit(uint32_t *w, uint2 f) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t fb = ((j < 4 ? f.x : f.y) >> (8 * (j & 3))) & 0xffu;
    if (fb) w[j >> 1] &= (j & 1) ? 0x0000ffffu : 0xffff0000u;
  }
}

template <int DT, bool ASYM, int L, bool ZERO>
__global__ void __launch_bounds__(kStreamThreads, 2)
    group_quant_tma(const void *__restrict__ x, int64_t n, int64_t n_units, int64_t n_units_pad,
                    FastDiv dc, const uint8_t *__restrict__ zflag,
                    uint32_t *__restrict__ codes, uint16_t *__restrict__ scales,
                    uint16_t *__restrict__ offsets, uint32_t *__restrict__ err) {
  pdl_entry();
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  constexpr int EB = Loader<DT>::kBytes;
  constexpr int kTileElems = kTileBytes / EB;
  constexpr int kTileUnits = kTileElems / 8;
  static_assert(kTileUnits % (kConsumerWarps * 32) == 0, "uniform consumer trip count");
  const int64_t n_tiles = (n + kTileElems - 1) / kTileElems;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {  // ---- producer: one elected lane drives the TMA engine
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        mbar_wait(&empty[stage], phase ^ 1);
        const int64_t e0 = t * kTileElems;
        const int64_t left = n - e0;
        const uint32_t bytes = static_cast<uint32_t>((left < kTileElems ? left : kTileElems) * EB);
        mbar_expect_tx(&full[stage], bytes);
        bulk_g2s(smem + stage * kTileBytes, static_cast<const char *>(x) + e0 * EB, bytes, &full[stage]);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // ---- consumers
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    mbar_wait(&full[stage], phase);
    const unsigned char *tile = smem + stage * kTileBytes;
    const int64_t u0 = t * kTileUnits;
#pragma unroll 1
    for (int j = threadIdx.x; j < kTileUnits; j += kConsumerWarps * 32) {
      const int64_t u = u0 + j;
      const bool act = u < n_units;
      uint4 hv = act ? smem_load8<DT>(tile, j) : make_uint4(0, 0, 0, 0);
      uint32_t w[4] = {hv.x, hv.y, hv.z, hv.w};
      if (ZERO && act) {
        const uint32_t e = static_cast<uint32_t>(u * 8);
        const uint32_t r = fdiv_u32(e, dc);
        const uint32_t c = e - r * dc.d;
        const uint2 f = __ldg(reinterpret_cast<const uint2 *>(zflag + c));
        if ((f.x | f.y) != 0) stream_zero_hit(w, f);
      }
      uint16_t s_bits, o_bits = 0;
      bool bad;
      if (ASYM) {
        uint32_t vmax = 0xFC00FC00u, vmin = 0x7C007C00u;
        if (act) {
          vmax = hmax2_nan(hmax2_nan(w[0], w[1]), hmax2_nan(w[2], w[3]));
          vmin = hmin2_nan(hmin2_nan(w[0], w[1]), hmin2_nan(w[2], w[3]));
        }
#pragma unroll
        for (int o = 1; o < L; o <<= 1) {
          vmax = hmax2_nan(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
          vmin = hmin2_nan(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        }
        vmax = hmax2_nan(vmax, __funnelshift_l(vmax, vmax, 16));
        vmin = hmin2_nan(vmin, __funnelshift_l(vmin, vmin, 16));
        const uint32_t hi = vmax & 0xffffu, lo = vmin & 0xffffu;
        bad = ((hi & 0x7fffu) >= 0x7c00u) || ((lo & 0x7fffu) >= 0x7c00u);
        asym_params(hi, lo, o_bits, s_bits);
      } else {
        uint32_t m = 0;
        if (act) {
          m = __vmaxu2(__vmaxu2(w[0] & 0x7fff7fffu, w[1] & 0x7fff7fffu),
                       __vmaxu2(w[2] & 0x7fff7fffu, w[3] & 0x7fff7fffu));
        }
#pragma unroll
        for (int o = 1; o < L; o <<= 1) m = __vmaxu2(m, __shfl_xor_sync(0xffffffffu, m, o));
        const uint32_t top = max(m & 0xffffu, m >> 16);
        bad = top >= 0x7c00u;
        s_bits = sym_scale_bits(top);
      }
      if ((lane & (L - 1)) == 0 && u < n_units_pad) {
        const int64_t grp = u / L;
        if (bad) raise_err(err, ADC_ERR_NONFINITE);
        scales[grp] = s_bits;
        if (ASYM) offsets[grp] = o_bits;
      }
      if (act) {
        uint32_t tb[8];
        if (ASYM) {
          const QParams q = make_qparams(s_bits, o_bits);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            tb[2 * i] = asym_tbits(__low2float(*reinterpret_cast<const __half2 *>(&w[i])), q);
            tb[2 * i + 1] = asym_tbits(__high2float(*reinterpret_cast<const __half2 *>(&w[i])), q);
          }
        } else if (s_bits >= 0x0400u) {
          const float sc = h2f(s_bits), inv = rcp_approx(sc);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            tb[2 * i] = sym_tbits(__low2float(*reinterpret_cast<const __half2 *>(&w[i])), sc, inv);
            tb[2 * i + 1] = sym_tbits(__high2float(*reinterpret_cast<const __half2 *>(&w[i])), sc, inv);
          }
        } else {
          const float s0 = h2f(s_bits), sc = s0 == 0.f ? 1.f : s0, inv = rcp_approx(sc);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            tb[2 * i] = sym_tbits_clip2(__low2float(*reinterpret_cast<const __half2 *>(&w[i])), sc, inv);
            tb[2 * i + 1] = sym_tbits_clip2(__high2float(*reinterpret_cast<const __half2 *>(&w[i])), sc, inv);
          }
        }
        __stcs(codes + u, pack8_tbits(tb));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1;
    }
  }
}

#define ADC_DT_SWITCH(dt, DT, ...)                                   \
  switch (dt) {                                                      \
    case ADC_F32: { constexpr int DT = ADC_F32; __VA_ARGS__; break; }  \
    case ADC_BF16: { constexpr int DT = ADC_BF16; __VA_ARGS__; break; } \
    case ADC_F16: { constexpr int DT = ADC_F16; __VA_ARGS__; break; }  \
    default: return -1;                                              \
  }

#define ADC_L_SWITCH(l, L, ...)                         \
  switch (l) {                                          \
    case 1: { constexpr int L = 1; __VA_ARGS__; break; }  \
    case 2: { constexpr int L = 2; __VA_ARGS__; break; }  \
    case 4: { constexpr int L = 4; __VA_ARGS__; break; }  \
    case 8: { constexpr int L = 8; __VA_ARGS__; break; }  \
    case 16: { constexpr int L = 16; __VA_ARGS__; break; } \
    case 32: { constexpr int L = 32; __VA_ARGS__; break; } \
    default: return -1;                                 \
  }

template <int DT, bool ASYM, int L, bool ZERO>
static int launch_one(const Ctx &c, const void *x, int64_t n, int64_t n_units, int64_t n_units_pad,
                      FastDiv dc, const uint8_t *zflag, uint32_t *codes, uint16_t *scales,
                      uint16_t *offsets, uint32_t *err) {
  static bool configured = false;  // per template instance
  if (!configured) {
    if (cudaFuncSetAttribute(group_quant_tma<DT, ASYM, L, ZERO>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem) != cudaSuccess)
      return -2;
    configured = true;
  }
  constexpr int kTileElems = kTileBytes / Loader<DT>::kBytes;
  const int64_t n_tiles = (n + kTileElems - 1) / kTileElems;
  int64_t grid = static_cast<int64_t>(c.num_sms) * 2;
  if (grid > n_tiles) grid = n_tiles;
  launch_k(group_quant_tma<DT, ASYM, L, ZERO>, static_cast<int>(grid), kStreamThreads, kStreamSmem, c.stream, 
      x, n, n_units, n_units_pad, dc, zflag, codes, scales, offsets, err);
  note_launches(1);
  return 0;
}

int launch_group_compress_tma(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                              int L, bool asym, const uint8_t *zero_flag, uint8_t *codes,
                              uint16_t *scales, uint16_t *offsets, uint32_t *err) {
  const int64_t n = rows * cols;
  const int64_t n_units = n / 8;
  const int64_t n_units_pad = (n_units + L - 1) / L * L;
  const FastDiv dc = make_fastdiv(static_cast<uint32_t>(cols));
  uint32_t *c32 = reinterpret_cast<uint32_t *>(codes);
  int rc = 0;
  ADC_DT_SWITCH(dt, DT, ADC_L_SWITCH(L, LL, {
    if (asym)
      rc = launch_one<DT, true, LL, false>(c, x, n, n_units, n_units_pad, dc, nullptr, c32, scales,
                                           offsets, err);
    else if (zero_flag)
      rc = launch_one<DT, false, LL, true>(c, x, n, n_units, n_units_pad, dc, zero_flag, c32, scales,
                                           nullptr, err);
    else
      rc = launch_one<DT, false, LL, false>(c, x, n, n_units, n_units_pad, dc, nullptr, c32, scales,
                                            nullptr, err);
  }));
  return rc;
}

}  // namespace adc
