// K1/K2 (symmetric / asymmetric group int4) compress + decompress, the
// outlier-zeroing variant used by K4, and the generic any-shape fallbacks.
//
// Reference: _quantize (codec.py:216-242), quantize_symmetric (:245-252),
// quantize_asymmetric (:255-258), dequantize (:261-286).
//
// Fast path layout: one thread owns 8 consecutive elements ("unit"): one
// 128-bit load (bf16/f16; two for f32), one 32-bit store of 8 packed nibbles.
// A group of g = 8*L elements is owned by L adjacent lanes of a warp and
// reduced with L-wide xor shuffles; every lane derives the group's scale
// itself (no broadcast), lane 0 of the group stores it.
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "quant.cuh"

namespace adc {

__device__ __forceinline__ uint32_t fastdiv(uint32_t n, const FastDiv &f) {
  return static_cast<uint32_t>((static_cast<uint64_t>(n) * f.m) >> f.p);
}

// Zero the flagged channels of 8 consecutive elements (one row segment,
// codec.py:328-329).  The flag bytes of the segment are fetched together with
// the data (zero_flags8) so their latency overlaps the loads; the original
// values of flagged channels go to the (k, rows) side buffer from dedicated
// gather CTAs (OutlierSide), not from here: storing them here scattered
// 2-byte writes across k rows of the buffer and stalled the quantiser on the
// store queue (ncu, r1).
// e is a multiple of 8 and cols % 8 == 0, so the column is 8 * ((e / 8) mod
// (cols / 8)): dc divides by cols / 8, exact for e / 8 < 2^31 (n < 2^34).
__device__ __forceinline__ uint2 zero_flags8(int64_t e, const FastDiv &dc,
                                             const uint8_t *__restrict__ zflag) {
  const uint32_t e8 = static_cast<uint32_t>(e >> 3);
  const uint32_t c8 = e8 - fastdiv(e8, dc) * dc.d;
  return __ldg(reinterpret_cast<const uint2 *>(zflag) + c8);
}
// Side-buffer gather for the outlier-separated scheme (codec.py:331-341):
// val[rank][r] = f16(x[r, idx[rank]]).  Run by the first n_gather CTAs of the
// quantising launch, right after the column statistics, while x is still in
// L2; threads run along rows (coalesced stores), 8 ranks per thread with
// their loads issued together.
struct OutlierSide {
  const uint32_t *idx;
  const int32_t *k_dev;
  int64_t k_cap, rows, cols;
  uint16_t *val;
  int n_gather;  // leading CTAs that gather (0: none)
  const uint32_t *requant;  // non-null: quantise only if *requant != 0 (speculation missed)
  int tail_gather;  // 1: every quantising CTA gathers after its units (no leading gather CTAs)
};
constexpr int kGatherRanks = 8;

template <int DT>
__device__ __forceinline__ void gather_side(const void *__restrict__ x, const OutlierSide &o,
                                            int64_t cta, int64_t n_ctas) {
  const int64_t k = min(static_cast<int64_t>(*o.k_dev), o.k_cap);
  const int64_t row_blocks = (o.rows + kThreads - 1) / kThreads;
  const int64_t items = row_blocks * ((k + kGatherRanks - 1) / kGatherRanks);
  for (int64_t it = cta; it < items; it += n_ctas) {
    const int64_t rk0 = (it / row_blocks) * kGatherRanks;
    const int64_t r = (it % row_blocks) * kThreads + threadIdx.x;
    if (r >= o.rows) continue;
    uint16_t v[kGatherRanks];
#pragma unroll
    for (int j = 0; j < kGatherRanks; ++j)
      v[j] = rk0 + j < k ? Loader<DT>::load1(x, r * o.cols + __ldg(o.idx + rk0 + j)) : 0;
#pragma unroll
    for (int j = 0; j < kGatherRanks; ++j)
      if (rk0 + j < k) o.val[(rk0 + j) * o.rows + r] = v[j];
  }
}

__device__ __forceinline__ uint32_t bmax2_nan(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmax2_nan(*reinterpret_cast<__nv_bfloat162 *>(&a), *reinterpret_cast<__nv_bfloat162 *>(&b));
  return *reinterpret_cast<uint32_t *>(&r);
}
__device__ __forceinline__ uint32_t bmin2_nan(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmin2_nan(*reinterpret_cast<__nv_bfloat162 *>(&a), *reinterpret_cast<__nv_bfloat162 *>(&b));
  return *reinterpret_cast<uint32_t *>(&r);
}

// Exact asymmetric code of one element (h = its f16 value) for the elements
// whose fast quotient fell within the tie margin -- frequent for bf16 data,
// whose few mantissa bits make exact half-integer quotients common.
//   d = h - o with its TwoSum error (non-zero: a tiny element against a
//   large offset -> float64, as codec.py:223-231);
//   r = Markstein-refined d/s; within 2^-20 of a half-integer b the exact
//   residual d - b*s (one FMA, exact here) decides, ties to even.
__device__ __forceinline__ int asym_exact_code(float h, float s, float inv, float o) {
  const float d = h - o;
  const float bb = d - h;
  const float err = (h - (d - bb)) + (-o - bb);
  if (err != 0.f) {
    const double r = rint((static_cast<double>(h) - static_cast<double>(o)) / static_cast<double>(s));
    return static_cast<int>(fmin(fmax(r, -8.0), 7.0));
  }
  const float r0 = d * inv;
  const float r1 = fmaf(fmaf(-r0, s, d), inv, r0);
  const float c = (r1 + kMagic) - kMagic;  // RNE integer
  const float fr = r1 - c;
  int code = static_cast<int>(c);
  if (fabsf(fabsf(fr) - 0.5f) < 0x1p-20f) {
    const float bnd = c + (fr > 0.f ? 0.5f : -0.5f);  // nearest half-integer
    const float res = fmaf(-bnd, s, d);               // exact sign of q - bnd
    const int up = static_cast<int>(bnd + 0.5f), dn = up - 1;
    code = res > 0.f ? up : (res < 0.f ? dn : ((up & 1) == 0 ? up : dn));  // ties to even
  }
  return min(max(code, -8), 7);
}

// Word j (runtime) of a unit held in registers: a selp tree, so the unit
// stays in registers (an indexed access would go through local memory).
__device__ __forceinline__ uint32_t selp_u32(bool c, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\tselp.b32 %0, %1, %2, p;\n\t}"
      : "=r"(r) : "r"(a), "r"(b), "r"(static_cast<uint32_t>(c)));
  return r;
}
template <int NW>
__device__ __forceinline__ uint32_t mux_word(const uint32_t *w, int j) {
  if (NW == 4) {
    const uint32_t a = selp_u32(j & 1, w[1], w[0]), b = selp_u32(j & 1, w[3], w[2]);
    return selp_u32(j & 2, b, a);
  } else if (NW == 8) {
    const uint32_t a = selp_u32(j & 1, w[1], w[0]), b = selp_u32(j & 1, w[3], w[2]);
    const uint32_t c = selp_u32(j & 1, w[5 % NW], w[4 % NW]), d = selp_u32(j & 1, w[7 % NW], w[6 % NW]);
    const uint32_t ab = selp_u32(j & 2, b, a), cd = selp_u32(j & 2, d, c);
    return selp_u32(j & 4, cd, ab);
  } else {
    const uint32_t lo = mux_word<8>(w, j & 7), hi = mux_word<8>(w + (NW > 8 ? 8 : 0), j & 7);
    return selp_u32(j & 8, hi, lo);
  }
}

// Fast group kernel: a lane owns EPL (8 or 16) consecutive elements, a group
// of g = EPL*L elements is owned by L adjacent lanes; U units per lane are
// loaded before any is processed (memory-level parallelism).
template <int DT, bool ASYM, int L, bool ZERO, int EPL, int U>
__global__ void __launch_bounds__(kThreads, ((ASYM && EPL == 32) || EPL * U >= 64) ? 3 : 4)
    group_quant_fast(const void *__restrict__ x, int64_t n_units, int64_t n_units_pad, FastDiv dc,
                     const uint8_t *__restrict__ zflag, OutlierSide side,
                     uint32_t *__restrict__ codes, uint16_t *__restrict__ scales,
                     uint16_t *__restrict__ offsets, uint32_t *__restrict__ err) {
  if (!ZERO) pdl_entry();
  constexpr int NW = EPL / 2;  // 16-bit pairs per unit
  constexpr int NC = EPL / 8;  // packed code words per unit
  using R = Raw<DT>;
  constexpr bool BF = R::kBf16;
  int64_t cta = blockIdx.x, n_ctas = gridDim.x;
  // ZERO runs as a programmatic dependent of the column statistics
  // (launch_k_dep): the first units of x are loaded before the wait (x is an
  // input the statistics kernel only reads), the flags, the outlier indices
  // and k after it
  uint32_t wn[U][NW];
  uint2 zfn[U][NC];
  auto fetch_x = [&](int64_t b) {
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = b + k * kThreads + threadIdx.x;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (u < n_units) v = R::template load8<false>(x, u * EPL + 8 * q);
        wn[k][4 * q] = v.x;
        wn[k][4 * q + 1] = v.y;
        wn[k][4 * q + 2] = v.z;
        wn[k][4 * q + 3] = v.w;
      }
    }
  };
  auto fetch_flags = [&](int64_t b) {
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = b + k * kThreads + threadIdx.x;
#pragma unroll
      for (int q = 0; q < NC; ++q)
        zfn[k][q] = u < n_units ? zero_flags8(u * EPL + 8 * q, dc, zflag) : make_uint2(0, 0);
    }
  };
  bool pre = false;  // the first iteration's x units are in wn
  if (ZERO) {
    const int64_t qc = cta - side.n_gather;
    if (qc >= 0 && qc * kThreads * U < n_units_pad) {
      fetch_x(qc * kThreads * U);
      pre = true;
    }
    pdl_wait();
    pdl_trigger();
    if (cta < side.n_gather) {
      gather_side<DT>(x, side, cta, side.n_gather);
      return;
    }
    cta -= side.n_gather;
    n_ctas -= side.n_gather;
    // the speculative column-statistics kernel already wrote codes / scales
    // with the predicted channel set; re-quantise only if it missed
    if (side.requant && __ldcg(side.requant) == 0u) {
      if (side.tail_gather) gather_side<DT>(x, side, cta, n_ctas);
      return;
    }
  }
  const int64_t step = n_ctas * kThreads * U;
  // asymmetric at 32 elements per lane: the next iteration's loads are issued
  // before this one is processed (software pipeline), so every warp keeps a
  // unit in flight while it computes (80 registers, 3 CTAs per SM)
  constexpr bool PIPE = ASYM && EPL == 32;  // measured: asym 79.3 -> 77.5 us, sym / outlier slower
  auto fetch = [&](int64_t b) {
    fetch_x(b);
    if (ZERO) fetch_flags(b);
  };
  if (PIPE && cta * kThreads * U < n_units_pad) fetch(cta * kThreads * U);
  for (int64_t base = cta * kThreads * U; base < n_units_pad; base += step) {
    if (!PIPE) {
      if (pre) {
        fetch_flags(base);
        pre = false;
      } else {
        fetch(base);
      }
    }
    uint32_t w[U][NW];
    uint2 zf[U][NC];
#pragma unroll
    for (int k = 0; k < U; ++k) {
#pragma unroll
      for (int i = 0; i < NW; ++i) w[k][i] = wn[k][i];
#pragma unroll
      for (int q = 0; q < NC; ++q) zf[k][q] = zfn[k][q];
    }
    if (PIPE && base + step < n_units_pad) fetch(base + step);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      const bool act = u < n_units;
      if (ZERO) {
#pragma unroll
        for (int q = 0; q < NC; ++q) zero_apply8(&w[k][4 * q], zf[k][q]);
      }
      uint16_t s_bits, o_bits = 0;
      bool bad, native = true;
      if (ASYM) {
        // packed max/min (NaN-propagating) in the input's own 16-bit format
        uint32_t vmax = BF ? 0xFF80FF80u : 0xFC00FC00u, vmin = BF ? 0x7F807F80u : 0x7C007C00u;
        if (act) {
          vmax = w[k][0];
          vmin = w[k][0];
#pragma unroll
          for (int i = 1; i < NW; ++i) {
            vmax = BF ? bmax2_nan(vmax, w[k][i]) : hmax2_nan(vmax, w[k][i]);
            vmin = BF ? bmin2_nan(vmin, w[k][i]) : hmin2_nan(vmin, w[k][i]);
          }
        }
#pragma unroll
        for (int o = 1; o < L; o <<= 1) {
          const uint32_t a = __shfl_xor_sync(0xffffffffu, vmax, o), b = __shfl_xor_sync(0xffffffffu, vmin, o);
          vmax = BF ? bmax2_nan(vmax, a) : hmax2_nan(vmax, a);
          vmin = BF ? bmin2_nan(vmin, b) : hmin2_nan(vmin, b);
        }
        const uint32_t smax = __funnelshift_l(vmax, vmax, 16), smin = __funnelshift_l(vmin, vmin, 16);
        vmax = BF ? bmax2_nan(vmax, smax) : hmax2_nan(vmax, smax);
        vmin = BF ? bmin2_nan(vmin, smin) : hmin2_nan(vmin, smin);
        uint32_t hi = vmax & 0xffffu, lo = vmin & 0xffffu;
        if (BF) {
          hi = bf16_bits_to_f16_bits(hi);  // f16 rounding is monotone: f16(max) = max(f16)
          lo = bf16_bits_to_f16_bits(lo);
        }
        bad = ((hi & 0x7fffu) >= 0x7c00u) || ((lo & 0x7fffu) >= 0x7c00u);
        asym_params(hi, lo, o_bits, s_bits);
      } else {
        uint32_t m = 0;
        if (act) {
#pragma unroll
          for (int i = 0; i < NW; ++i) m = __vmaxu2(m, w[k][i] & 0x7fff7fffu);
        }
        m = warp_max_u2<L>(m);
        const uint32_t top = max(m & 0xffffu, m >> 16);
        if (BF) {
          bad = top >= 0x4780u;       // >= 65536 rounds to f16 inf (also inf/NaN)
          native = top >= 0x3900u;    // top >= 2^-13: scale >= 2^-16, tiny-value rounding is code-neutral
          s_bits = sym_scale_bits(bf16_bits_to_f16_bits(top));
        } else {
          bad = top >= 0x7c00u;
          s_bits = sym_scale_bits(top);
        }
      }
      const int64_t grp = u / L;
      if ((threadIdx.x & (L - 1)) == 0 && u < n_units_pad) {
        if (bad) raise_err(err, ADC_ERR_NONFINITE);
        scales[grp] = s_bits;
        if (ASYM) offsets[grp] = o_bits;
      }
      if (!act) continue;
      uint32_t t[EPL];
      uint32_t fix = 0;  // elements whose fast quotient is within the tie margin
      if (ASYM) {
        const QParams q = make_qparams(s_bits, o_bits);
        // r = RN(x*inv - RN(o*inv)) (one FFMA) is within 2^-19 + |o*inv|*2^-23
        // of the exact quotient (x - o)/s of the f16 value (inv: 1-ulp
        // reciprocal); for bf16 the native x differs from f16(x) by <= 2^-25
        // (tiny values only), i.e. by <= 2^-25/s in the quotient.  Elements
        // within that margin (doubled) of a half-integer are redone exactly.
        const float oi = q.o * q.inv;
        const float thr = 0.5f - (0x1p-17f + fabsf(oi) * 0x1p-22f + (BF ? 0x1p-25f * q.inv : 0.f));
        // no clips here: the codes saturate to [-8, 7] when packed
        // (pack8_tbits_sat); an unclipped quotient beyond the range only
        // rounds to a code the saturation maps to the clipped one, and a
        // near-tie flagged there is redone exactly like any other
        // two elements per FFMA2 / FADD2; rounding residuals |e| beyond thr
        // mark the elements redone exactly (frequent for bf16 data, whose
        // coarse mantissas make exact half-integer quotients common)
        const uint64_t inv2 = f2_pack(q.inv, q.inv), noi2 = f2_pack(-oi, -oi);
        const uint64_t mg2 = f2_pack(kMagic8, kMagic8);
        // the test |e| > thr as the sign of fma(e, e, -t2) (exact sign; t2 <
        // thr^2, so every near tie is caught, plus at most a few elements
        // just inside the margin, which the exact pass recomputes): one
        // FFMA2 per pair on the FMA pipe, then one funnel shift per element
        // pushes the sign into the mask (bit-reversed and inverted once)
        const float t2 = thr * thr * (1.f - 0x1p-20f);
        const uint64_t nt2 = f2_pack(-t2, -t2);
        uint32_t signs = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          const uint64_t r2 = f2_fma(f2_pack(R::lo(w[k][i]), R::hi(w[k][i])), inv2, noi2);
          const uint64_t tv2 = f2_add(r2, mg2);
          const uint64_t e2 = f2_sub(r2, f2_sub(tv2, mg2));
          float dl, dh, tl, th;
          f2_unpack(f2_fma(e2, e2, nt2), dl, dh);
          signs = __funnelshift_l(__float_as_uint(dl), signs, 1);
          signs = __funnelshift_l(__float_as_uint(dh), signs, 1);
          f2_unpack(tv2, tl, th);
          t[2 * i] = __float_as_uint(tl);
          t[2 * i + 1] = __float_as_uint(th);
        }
        fix = ~__brev(signs) >> (32 - EPL);
      } else if (!BF || native) {
        if (s_bits >= 0x0400u) {  // normal scale: upper clip only
          // correctly rounded h/s two lanes per FMUL2 / FFMA2 (Markstein),
          // RNE by the magic add, clip to 7 in the saturating pack
          const float sc = h2f(s_bits), inv = rcp_approx(sc);
          const uint64_t inv2 = f2_pack(inv, inv), ns2 = f2_pack(-sc, -sc), mg2 = f2_pack(kMagic8, kMagic8);
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            const uint64_t h2 = f2_pack(R::lo(w[k][i]), R::hi(w[k][i]));
            const uint64_t r0 = f2_mul(h2, inv2);
            const uint64_t r1 = f2_fma(f2_fma(r0, ns2, h2), inv2, r0);
            float tl, th;
            f2_unpack(f2_add(r1, mg2), tl, th);
            t[2 * i] = __float_as_uint(tl);  // upper clip: saturating pack
            t[2 * i + 1] = __float_as_uint(th);
          }
        } else {
          const float s0 = h2f(s_bits), sc = s0 == 0.f ? 1.f : s0, inv = rcp_approx(sc);
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            t[2 * i] = sym_tbits_clip2(R::lo(w[k][i]), sc, inv);
            t[2 * i + 1] = sym_tbits_clip2(R::hi(w[k][i]), sc, inv);
          }
        }
      } else {  // bf16 group with a tiny maximum: exact converting path
        unit_codes_exact<BF, NW>(w[k], h2f(s_bits), 0.f, false, t);
      }
      uint32_t cw[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) cw[q] = pack8_tbits_sat(t + 8 * q);
      if (ASYM) {
        const float sc = h2f(s_bits), so = h2f(o_bits);
        const float scd = sc == 0.f ? 1.f : sc, inv = rcp_approx(scd);
        // one near-tie element per lane per round, all lanes together: the
        // warp pays max(popcount(fix)) rounds (usually one) instead of one
        // divergent pass per element position
        while (__any_sync(__activemask(), fix != 0)) {
          if (fix) {
            const int i = __ffs(fix) - 1;
            fix &= fix - 1;
            const uint32_t word = mux_word<NW>(w[k], i >> 1);
            const uint32_t raw = (word >> (16 * (i & 1))) & 0xffffu;
            const int code = asym_exact_code(h2f(BF ? bf16_bits_to_f16_bits(raw) : raw), scd, inv, so);
            const uint32_t sh = 4 * (i & 7), nib = static_cast<uint32_t>(code) & 0xfu;
            const uint32_t m = ~(0xfu << sh), v = nib << sh;
#pragma unroll
            for (int q = 0; q < NC; ++q)
              if ((i >> 3) == q) cw[q] = (cw[q] & m) | v;
          }
        }
      }
      if (NC == 1) {
        codes[u] = cw[0];
      } else if (NC == 2) {
        *reinterpret_cast<uint2 *>(codes + 2 * u) = make_uint2(cw[0], cw[NC - 1]);
      } else {
        *reinterpret_cast<uint4 *>(codes + 4 * u) = make_uint4(cw[0], cw[1 % NC], cw[2 % NC], cw[3 % NC]);
      }
    }
  }
  if (ZERO && side.tail_gather) gather_side<DT>(x, side, cta, n_ctas);
}

template <int OT, bool ASYM, int L, int EPL, int U>
__global__ void __launch_bounds__(kThreads)
    group_dequant_fast(const uint32_t *__restrict__ codes, const uint16_t *__restrict__ scales,
                       const uint16_t *__restrict__ offsets, int64_t n_units, void *__restrict__ y) {
  pdl_entry();
  constexpr int NC = EPL / 8;
  const int64_t step = static_cast<int64_t>(gridDim.x) * kThreads * U;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads * U; base < n_units;
       base += step) {
    uint32_t w[U][NC];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      if (NC == 1) {
        w[k][0] = (u < n_units) ? __ldcs(codes + u) : 0u;
      } else {
        const uint2 v = (u < n_units) ? __ldcs(reinterpret_cast<const uint2 *>(codes) + u) : make_uint2(0, 0);
        w[k][0] = v.x;
        w[k][NC - 1] = v.y;
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t u = base + k * kThreads + threadIdx.x;
      if (u >= n_units) continue;
      const int64_t grp = u / L;
      const float s = h2f(__ldg(scales + grp));
      const float o = ASYM ? h2f(__ldg(offsets + grp)) : 0.f;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = deq<ASYM>(nib_code(w[k][q], j), s, o);
        Storer<OT>::store8(y, u * EPL + 8 * q, v);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// generic fallbacks: any group size (incl. PER_CHANNEL), any shape/alignment
// ---------------------------------------------------------------------------
template <int DT, bool ASYM>
__global__ void __launch_bounds__(kThreads)
    group_stats_generic(const void *__restrict__ x, int64_t n, int64_t g, int64_t n_groups,
                        bool pc, int64_t rows, int64_t cols, const uint8_t *__restrict__ zflag,
                        uint16_t *__restrict__ scales, uint16_t *__restrict__ offsets,
                        uint32_t *__restrict__ err) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + threadIdx.x / 32;
       j < n_groups; j += warps) {
    const int64_t count = pc ? rows : min(g, n - j * g);
    uint32_t amax = 0, kmax = 0, kmin = 0xffffu;
    bool bad = false;
    for (int64_t i = lane; i < count; i += 32) {
      const int64_t e = pc ? i * cols + j : j * g + i;
      uint32_t b = Loader<DT>::load1(x, e);
      bad |= (b & 0x7fffu) >= 0x7c00u;
      if (zflag && zflag[e % cols]) b = 0;
      amax = max(amax, b & 0x7fffu);
      kmax = max(kmax, f16_key(b));
      kmin = min(kmin, f16_key(b));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (bad) raise_err(err, ADC_ERR_NONFINITE);
      if (ASYM) {
        uint16_t o, s;
        asym_params(f16_unkey(kmax), f16_unkey(kmin), o, s);
        scales[j] = s;
        offsets[j] = o;
      } else {
        scales[j] = sym_scale_bits(amax);
      }
    }
  }
}

template <int DT, bool ASYM>
__global__ void __launch_bounds__(kThreads)
    group_quant_generic(const void *__restrict__ x, int64_t n, int64_t g, bool pc, int64_t rows,
                        int64_t cols, const uint8_t *__restrict__ zflag,
                        const uint16_t *__restrict__ scales, const uint16_t *__restrict__ offsets,
                        uint8_t *__restrict__ codes) {
  pdl_entry();
  const int64_t nbytes = (n + 1) / 2;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; b < nbytes;
       b += static_cast<int64_t>(gridDim.x) * kThreads) {
    uint32_t byte = 0;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t p = 2 * b + half;  // position in the code stream
      if (p >= n) break;
      int64_t r, c, grp;
      if (pc) {
        c = p / rows;
        r = p - c * rows;
        grp = c;
      } else {
        r = p / cols;
        c = p - r * cols;
        grp = p / g;
      }
      uint32_t hb = Loader<DT>::load1(x, r * cols + c);
      if (zflag && zflag[c]) hb = 0;
      QParams q = make_qparams(scales[grp], ASYM ? offsets[grp] : 0);
      int code = quant_code<ASYM>(h2f(hb), q);
      byte |= (static_cast<uint32_t>(code) & 0xfu) << (4 * half);
    }
    codes[b] = static_cast<uint8_t>(byte);
  }
}

// Stand-alone side-buffer gather (generic path and the TMA variant).
template <int DT>
__global__ void __launch_bounds__(kThreads)
    outlier_gather(const void *__restrict__ x, OutlierSide side) {
  pdl_entry();
  gather_side<DT>(x, side, blockIdx.x, gridDim.x);
}

template <int OT, bool ASYM>
__global__ void __launch_bounds__(kThreads)
    group_dequant_generic(const uint8_t *__restrict__ codes, const uint16_t *__restrict__ scales,
                          const uint16_t *__restrict__ offsets, int64_t n, int64_t g, bool pc,
                          int64_t rows, int64_t cols, void *__restrict__ y) {
  pdl_entry();
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * kThreads) {
    const int64_t r = e / cols, c = e - r * cols;
    const int64_t p = pc ? c * rows + r : e;
    const int64_t grp = pc ? c : p / g;
    const uint32_t nib = (codes[p >> 1] >> ((p & 1) * 4)) & 0xfu;
    const float code = __int_as_float(0x4B400000 | (nib ^ 8u)) - (kMagic + 8.f);
    const float s = h2f(scales[grp]);
    const float o = ASYM ? h2f(offsets[grp]) : 0.f;
    Storer<OT>::store1(y, e, deq<ASYM>(code, s, o));
  }
}

template <int OT>
__global__ void __launch_bounds__(kThreads)
    outlier_scatter(const uint32_t *__restrict__ idx, const uint16_t *__restrict__ val,
                    const int32_t *__restrict__ k_dev, int64_t k_cap, int64_t rows, int64_t cols,
                    void *__restrict__ y) {
  pdl_entry();
  // blockIdx.y walks the ranks, x the rows: no division, coalesced side-buffer reads
  const int64_t k = min(static_cast<int64_t>(*k_dev), k_cap);
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
    const int64_t c = __ldg(idx + j);
    const uint16_t *vj = val + j * rows;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * kThreads)
      Storer<OT>::store1(y, r * cols + c, h2f(__ldg(vj + r)));
  }
}

// Outlier-separated decompress in ONE launch (codec.py:276-285).  Each CTA
// owns a TILE of the row-major output (T elements): it dequantises the tile's
// 8-element units into shared memory, overwrites the flagged channels of the
// rows the tile spans there (the side-buffer values were requested before the
// dequantisation, so their latency overlaps it), and streams the finished
// tile out with full 128-bit stores -- no 2-byte scatter into global memory,
// hence no partial-sector writes at any output size.
template <int OT>
__device__ __forceinline__ void put8_shared(unsigned char *t, const float *v) {
  if constexpr (OT == ADC_F32) {
    reinterpret_cast<uint4 *>(t)[0] = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                                 __float_as_uint(v[2]), __float_as_uint(v[3]));
    reinterpret_cast<uint4 *>(t)[1] = make_uint4(__float_as_uint(v[4]), __float_as_uint(v[5]),
                                                 __float_as_uint(v[6]), __float_as_uint(v[7]));
  } else if constexpr (OT == ADC_BF16) {
    *reinterpret_cast<uint4 *>(t) = make_uint4(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]),
                                               pack_bf2(v[4], v[5]), pack_bf2(v[6], v[7]));
  } else {
    *reinterpret_cast<uint4 *>(t) = make_uint4(f32x2_to_h2(v[0], v[1]), f32x2_to_h2(v[2], v[3]),
                                               f32x2_to_h2(v[4], v[5]), f32x2_to_h2(v[6], v[7]));
  }
}

template <int OT>
__device__ __forceinline__ void put1_shared(unsigned char *t, float v) {
  if constexpr (OT == ADC_F32) *reinterpret_cast<float *>(t) = v;
  else if constexpr (OT == ADC_BF16) *reinterpret_cast<__nv_bfloat16 *>(t) = __float2bfloat16_rn(v);
  else *reinterpret_cast<__half *>(t) = __float2half_rn(v);
}

template <int OT, int L, int T>
__global__ void __launch_bounds__(kThreads)
    outlier_dequant_tiles(const uint32_t *__restrict__ codes, const uint16_t *__restrict__ scales,
                          int64_t rows, int64_t cols, int64_t n, const uint32_t *__restrict__ idx,
                          const uint16_t *__restrict__ val, const int32_t *__restrict__ k_dev, int k_cap,
                          void *__restrict__ y) {
  constexpr int OSZ = OT == ADC_F32 ? 4 : 2;
  constexpr int UPT = T / 8 / kThreads;  // 8-element units per thread
  constexpr int PF = 2;                  // side-buffer pairs prefetched per thread
  __shared__ __align__(16) unsigned char tile[T * OSZ];
  pdl_entry();
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * T;
  const int te = static_cast<int>(min(n - e0, static_cast<int64_t>(T)));  // multiple of 8
  const int kk = min(__ldg(k_dev), k_cap);
  uint32_t w[UPT];
#pragma unroll
  for (int q = 0; q < UPT; ++q) {
    const int lu = q * kThreads + threadIdx.x;
    w[q] = lu * 8 < te ? __ldcs(codes + (e0 >> 3) + lu) : 0u;
  }
  const int64_t ra = e0 / cols;
  const int nr = static_cast<int>((e0 + te - 1) / cols - ra + 1);
  const int pairs = kk * nr;
  uint32_t pc[PF];
  uint16_t pv[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int p = threadIdx.x + i * kThreads;
    if (p < pairs) {
      const int j = p / nr, rr = p - j * nr;
      pc[i] = __ldg(idx + j);
      pv[i] = __ldg(val + static_cast<int64_t>(j) * rows + ra + rr);
    }
  }
#pragma unroll
  for (int q = 0; q < UPT; ++q) {
    const int lu = q * kThreads + threadIdx.x;
    if (lu * 8 >= te) continue;
    const float s = h2f(__ldg(scales + ((e0 >> 3) + lu) / L));
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = deq<false>(nib_code(w[q], j), s, 0.f);
    put8_shared<OT>(tile + lu * 8 * OSZ, v);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int p = threadIdx.x + i * kThreads;
    if (p < pairs) {
      const int j = p / nr, rr = p - j * nr;
      const int64_t e = (ra + rr) * cols + pc[i] - e0;
      if (e >= 0 && e < te) put1_shared<OT>(tile + e * OSZ, h2f(pv[i]));
    }
  }
  for (int p = threadIdx.x + PF * kThreads; p < pairs; p += kThreads) {
    const int j = p / nr, rr = p - j * nr;
    const int64_t e = (ra + rr) * cols + __ldg(idx + j) - e0;
    if (e >= 0 && e < te) put1_shared<OT>(tile + e * OSZ, h2f(__ldg(val + static_cast<int64_t>(j) * rows + ra + rr)));
  }
  __syncthreads();
  char *dst = static_cast<char *>(y) + e0 * OSZ;
  for (int off = threadIdx.x * 16; off < te * OSZ; off += kThreads * 16)
    st_stream16(dst + off, *reinterpret_cast<const uint4 *>(tile + off));
}

// Outlier overwrite after the plain dequantisation (codec.py:284-285), one
// thread per (rank, row) rewriting the whole 32-byte sector that holds the
// flagged element: 16 dequantised values (their 128-group's scale; sectors
// never straddle a group) with the stored float16 values of every flagged
// channel in that sector.  Full-sector stores avoid the read-modify-write a
// 2-byte scatter costs once the output has left L2 (k x rows partial sectors).
// The first rank of a sector owns it.  Ranks on grid.y, rows on grid.x.
template <int OT, int L>
__global__ void __launch_bounds__(kThreads)
    outlier_patch16(const uint32_t *__restrict__ codes, const uint16_t *__restrict__ scales,
                    const uint32_t *__restrict__ idx, const uint16_t *__restrict__ val,
                    const int32_t *__restrict__ k_dev, int64_t k_cap, int64_t rows, int64_t cols,
                    void *__restrict__ y) {
  pdl_entry();
  constexpr int SE = 32 / Storer<OT>::kBytes;  // elements per 32-byte sector (16 bf16/f16, 8 f32)
  const int64_t k = min(static_cast<int64_t>(*k_dev), k_cap);
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
    const uint32_t c = __ldg(idx + j);
    const uint32_t sec = c / SE;
    if (j > 0 && __ldg(idx + j - 1) / SE == sec) continue;  // an earlier rank owns this sector
    int nj = 1;                                             // ranks in this sector: j .. j + nj - 1
    while (j + nj < k && nj < SE && __ldg(idx + j + nj) / SE == sec) ++nj;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * kThreads) {
      const int64_t e0 = r * cols + static_cast<int64_t>(sec) * SE;  // first element of the sector
      const int64_t u0 = e0 / 8;                                     // its first 8-element code word
      float v[16];
      const float sc = h2f(__ldg(scales + e0 / (8 * L)));
#pragma unroll
      for (int h = 0; h < SE / 8; ++h) {
        const uint32_t w = __ldg(codes + u0 + h);
#pragma unroll
        for (int q = 0; q < 8; ++q) v[8 * h + q] = deq<false>(nib_code(w, q), sc, 0.f);
      }
      for (int t = 0; t < nj; ++t) {
        const uint32_t cc = __ldg(idx + j + t) - sec * SE;
        const float hv = h2f(__ldg(val + (j + t) * rows + r));
#pragma unroll
        for (int q = 0; q < SE; ++q)
          if (q == static_cast<int>(cc)) v[q] = hv;
      }
#pragma unroll
      for (int h = 0; h < SE / 8; ++h) Storer<OT>::store8(y, e0 + 8 * h, v + 8 * h);
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
// 32 elements per lane (one 128-bit code store, the group's scale work
// amortised over twice the elements) vs 16; ADC_EPL=16 or
// adc_set_option("epl", 16) selects the 16-element kernels (A/B testing).
static std::atomic<int> g_epl{-1};
bool use_epl32() {
  int v = g_epl.load(std::memory_order_relaxed);
  if (v < 0) {
    const char *e = getenv("ADC_EPL");
    v = (e && e[0] == '1') ? 16 : 32;
    g_epl.store(v, std::memory_order_relaxed);
  }
  return v == 32;
}
void set_epl(int v) { g_epl.store(v == 16 ? 16 : 32, std::memory_order_relaxed); }

static inline int grid_for(const Ctx &c, int64_t work_items, int per_block) {
  int64_t need = (work_items + per_block - 1) / per_block;
  int64_t cap = static_cast<int64_t>(c.num_sms) * 8;
  if (need < 1) need = 1;
  return static_cast<int>(need < cap ? need : cap);
}

static inline bool aligned(const void *p, size_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

// Lanes per group for EPL elements per lane (0: no fast path).
static inline int lanes_for_group(int64_t g, int epl) {
  if (g < epl || g > 32 * epl || g % epl) return 0;
  const int64_t l = g / epl;
  return (l & (l - 1)) == 0 ? static_cast<int>(l) : 0;
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

constexpr int kUnroll = 2;
constexpr int kU32 = 1;  // units in flight per lane at 32 elements per lane
constexpr int kUD = 4;   // units in flight per lane in the 8-element dequantiser

// Gather work: (k_cap / 8) rank blocks x (rows / 256) row blocks, either up
// to one leading gather CTA per SM, or taken by the quantising CTAs after
// their units ("tail").  Leading CTAs hold slots the one-wave quantiser grid
// counts on, so its last CTAs start late: measured 147 -> 143 us at
// [131072, 1024] with the tail, but 19.5 -> 20.1 us at [8192, 1024] (the
// tail adds a dependent gather round trip to short kernels).  Default: tail
// from 2^26 elements; ADC_GATHER_TAIL=0/1 forces either.
static bool use_tail_gather(int64_t n) {
  const char *e = getenv("ADC_GATHER_TAIL");
  return e ? atoi(e) != 0 : n >= (int64_t{1} << 26);
}
static OutlierSide outlier_side(const Ctx &c, const uint32_t *idx, const int32_t *k_dev,
                                int64_t k_cap, int64_t rows, int64_t cols, uint16_t *val,
                                bool tail_ok = true) {
  OutlierSide o{idx, k_dev, k_cap, rows, cols, val, 0, nullptr, 0};
  if (k_cap <= 0 || !val || !idx || !k_dev) return o;
  if (tail_ok && use_tail_gather(rows * cols)) {
    o.tail_gather = 1;
    return o;
  }
  const int64_t items = ((rows + kThreads - 1) / kThreads) * ((k_cap + kGatherRanks - 1) / kGatherRanks);
  o.n_gather = static_cast<int>(items < c.num_sms ? items : c.num_sms);
  return o;
}

int launch_group_compress(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                          int64_t g, bool asym, const uint8_t *zero_flag, const uint32_t *idx, const int32_t *k_dev, uint16_t *outl_val,
                          int64_t k_cap, uint8_t *codes, uint16_t *scales, uint16_t *offsets,
                          uint32_t *err, const uint32_t *requant) {
  const int64_t n = rows * cols;
  const bool pc = (g == 0);
  const bool zero = zero_flag != nullptr;
  const bool zero_ok = !zero || (cols % 8 == 0 && n / 8 < (1ll << 31));
  const FastDiv dc = make_fastdiv(static_cast<uint32_t>(cols >= 8 ? cols / 8 : 1));  // zero_flags8
  OutlierSide side = outlier_side(c, idx, k_dev, zero ? k_cap : 0, rows, cols, outl_val);
  side.requant = zero ? requant : nullptr;
  int L = pc ? 0 : lanes_for_group(g, 32);
  if (L > 0 && use_epl32() && n % 32 == 0 && aligned(x, 16) && aligned(codes, 16) && zero_ok) {
    const int64_t n_units = n / 32;
    const int64_t n_units_pad = (n_units + L - 1) / L * L;
    const int grid = grid_for(c, n_units_pad, kThreads * kU32);
    uint32_t *codes32 = reinterpret_cast<uint32_t *>(codes);
    ADC_DT_SWITCH(dt, DT, ADC_L_SWITCH(L, LL, {
      if (asym) {
        launch_k(group_quant_fast<DT, true, LL, false, 32, kU32>, grid, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, nullptr, OutlierSide{}, codes32, scales, offsets, err), note_launches(1);
      } else if (zero && n < (int64_t{1} << 26)) {
        // a programmatic dependent of the column pass below 2^26 elements (x still in L2, the
        // statistics tail a large share); measured slower beyond: [131072,4096] 524 -> 557 us
        launch_k_dep(group_quant_fast<DT, false, LL, true, 32, kU32>, grid + side.n_gather, kThreads, 0, c.stream,
            x, n_units, n_units_pad, dc, zero_flag, side, codes32, scales, nullptr, err), note_launches(1);
      } else if (zero) {
        launch_k(group_quant_fast<DT, false, LL, true, 32, kU32>, grid + side.n_gather, kThreads, 0, c.stream,
            x, n_units, n_units_pad, dc, zero_flag, side, codes32, scales, nullptr, err), note_launches(1);
      } else {
        launch_k(group_quant_fast<DT, false, LL, false, 32, kU32>, grid, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, nullptr, OutlierSide{}, codes32, scales, nullptr, err), note_launches(1);
      }
    }));
    return 0;
  }
  L = pc ? 0 : lanes_for_group(g, 16);
  if (L > 0 && n % 16 == 0 && aligned(x, 16) && aligned(codes, 8) && zero_ok) {
    const int64_t n_units = n / 16;
    const int64_t n_units_pad = (n_units + L - 1) / L * L;
    const int grid = grid_for(c, n_units_pad, kThreads * kUnroll);
    uint32_t *codes32 = reinterpret_cast<uint32_t *>(codes);
    ADC_DT_SWITCH(dt, DT, ADC_L_SWITCH(L, LL, {
      if (asym) {
        launch_k(group_quant_fast<DT, true, LL, false, 16, kUnroll>, grid, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, nullptr, OutlierSide{}, codes32, scales, offsets, err), note_launches(1);
      } else if (zero) {
        launch_k_dep(group_quant_fast<DT, false, LL, true, 16, kUnroll>, grid + side.n_gather, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, zero_flag, side, codes32, scales, nullptr, err), note_launches(1);
      } else {
        launch_k(group_quant_fast<DT, false, LL, false, 16, kUnroll>, grid, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, nullptr, OutlierSide{}, codes32, scales, nullptr, err), note_launches(1);
      }
    }));
    return 0;
  }
  L = pc ? 0 : lanes_for_group(g, 8);
  if (L > 0 && n % 8 == 0 && aligned(x, 16) && aligned(codes, 4) && zero_ok) {
    const int64_t n_units = n / 8;
    const int64_t n_units_pad = (n_units + L - 1) / L * L;
    const int grid = grid_for(c, n_units_pad, kThreads * kUnroll);
    uint32_t *codes32 = reinterpret_cast<uint32_t *>(codes);
    ADC_DT_SWITCH(dt, DT, ADC_L_SWITCH(L, LL, {
      if (asym) {
        launch_k(group_quant_fast<DT, true, LL, false, 8, kUnroll>, grid, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, nullptr, OutlierSide{}, codes32, scales, offsets, err), note_launches(1);
      } else if (zero) {
        launch_k_dep(group_quant_fast<DT, false, LL, true, 8, kUnroll>, grid + side.n_gather, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, zero_flag, side, codes32, scales, nullptr, err), note_launches(1);
      } else {
        launch_k(group_quant_fast<DT, false, LL, false, 8, kUnroll>, grid, kThreads, 0, c.stream, 
            x, n_units, n_units_pad, dc, nullptr, OutlierSide{}, codes32, scales, nullptr, err), note_launches(1);
      }
    }));
    return 0;
  }
  // generic: per-group stats, then per-byte quantisation
  const int64_t n_groups = pc ? cols : (n + g - 1) / g;
  const int gs = grid_for(c, n_groups, kThreads / 32);
  const int gq = grid_for(c, (n + 1) / 2, kThreads);
  ADC_DT_SWITCH(dt, DT, {
    if (asym) {
      launch_k(group_stats_generic<DT, true>, gs, kThreads, 0, c.stream, 
          x, n, g, n_groups, pc, rows, cols, zero_flag, scales, offsets, err), note_launches(1);
      launch_k(group_quant_generic<DT, true>, gq, kThreads, 0, c.stream, x, n, g, pc, rows, cols,
                                                                    zero_flag, scales, offsets,
                                                                    codes), note_launches(1);
    } else {
      launch_k(group_stats_generic<DT, false>, gs, kThreads, 0, c.stream, 
          x, n, g, n_groups, pc, rows, cols, zero_flag, scales, nullptr, err), note_launches(1);
      launch_k(group_quant_generic<DT, false>, gq, kThreads, 0, c.stream, x, n, g, pc, rows, cols,
                                                                     zero_flag, scales, nullptr,
                                                                     codes), note_launches(1);
    }
  });
  if (zero_flag) return launch_outlier_gather(c, x, dt, idx, k_dev, k_cap, rows, cols, outl_val);
  return 0;
}

int launch_outlier_gather(const Ctx &c, const void *x, int dt, const uint32_t *idx,
                          const int32_t *k_dev, int64_t k_cap, int64_t rows, int64_t cols,
                          uint16_t *outl_val) {
  const OutlierSide side = outlier_side(c, idx, k_dev, k_cap, rows, cols, outl_val, false);
  if (side.n_gather == 0) return 0;
  ADC_DT_SWITCH(dt, DT, launch_k(outlier_gather<DT>, side.n_gather, kThreads, 0, c.stream, x, side),
                note_launches(1));
  return 0;
}

#define ADC_OT_SWITCH(ot, OT, ...)                                   \
  switch (ot) {                                                      \
    case ADC_F32: { constexpr int OT = ADC_F32; __VA_ARGS__; break; }  \
    case ADC_BF16: { constexpr int OT = ADC_BF16; __VA_ARGS__; break; } \
    case ADC_F16: { constexpr int OT = ADC_F16; __VA_ARGS__; break; }  \
    default: return -1;                                              \
  }

int launch_group_decompress(const Ctx &c, const uint8_t *codes, const uint16_t *scales,
                            const uint16_t *offsets, int64_t rows, int64_t cols, int64_t g,
                            bool asym, void *y, int ot) {
  const int64_t n = rows * cols;
  const bool pc = (g == 0);
  // 8 elements per lane measured faster than 16 for the store-bound inverse
  int L = pc ? 0 : lanes_for_group(g, 8);
  if (L > 0 && n % 8 == 0 && aligned(y, 16) && aligned(codes, 4)) {
    const int64_t n_units = n / 8;
    const uint32_t *codes32 = reinterpret_cast<const uint32_t *>(codes);
    // 4 units in flight per lane up to 64 M elements (measured: [8192,4096]
    // 16.2 -> 15.7 us, [8192,3072] 12.7 -> 11.9 us), 2 beyond (268 MB:
    // 57.3 us with 2 vs 62.9 us with 4)
    if (n_units <= (8ll << 20)) {
      const int grid = grid_for(c, n_units, kThreads * kUD);
      ADC_OT_SWITCH(ot, OT, ADC_L_SWITCH(L, LL, {
        if (asym)
          launch_k(group_dequant_fast<OT, true, LL, 8, kUD>, grid, kThreads, 0, c.stream,
                   codes32, scales, offsets, n_units, y), note_launches(1);
        else
          launch_k(group_dequant_fast<OT, false, LL, 8, kUD>, grid, kThreads, 0, c.stream,
                   codes32, scales, nullptr, n_units, y), note_launches(1);
      }));
    } else {
      const int grid = grid_for(c, n_units, kThreads * kUnroll);
      ADC_OT_SWITCH(ot, OT, ADC_L_SWITCH(L, LL, {
        if (asym)
          launch_k(group_dequant_fast<OT, true, LL, 8, kUnroll>, grid, kThreads, 0, c.stream,
                   codes32, scales, offsets, n_units, y), note_launches(1);
        else
          launch_k(group_dequant_fast<OT, false, LL, 8, kUnroll>, grid, kThreads, 0, c.stream,
                   codes32, scales, nullptr, n_units, y), note_launches(1);
      }));
    }
    return 0;
  }
  L = pc ? 0 : lanes_for_group(g, 16);
  if (L > 0 && n % 16 == 0 && aligned(y, 16) && aligned(codes, 8)) {
    const int64_t n_units = n / 16;
    const int grid = grid_for(c, n_units, kThreads * kUnroll);
    const uint32_t *codes32 = reinterpret_cast<const uint32_t *>(codes);
    ADC_OT_SWITCH(ot, OT, ADC_L_SWITCH(L, LL, {
      if (asym)
        launch_k(group_dequant_fast<OT, true, LL, 16, kUnroll>, grid, kThreads, 0, c.stream, 
            codes32, scales, offsets, n_units, y), note_launches(1);
      else
        launch_k(group_dequant_fast<OT, false, LL, 16, kUnroll>, grid, kThreads, 0, c.stream, 
            codes32, scales, nullptr, n_units, y), note_launches(1);
    }));
    return 0;
  }
  const int grid = grid_for(c, n, kThreads);
  ADC_OT_SWITCH(ot, OT, {
    if (asym)
      launch_k(group_dequant_generic<OT, true>, grid, kThreads, 0, c.stream, codes, scales, offsets, n,
                                                                       g, pc, rows, cols, y), note_launches(1);
    else
      launch_k(group_dequant_generic<OT, false>, grid, kThreads, 0, c.stream, codes, scales, nullptr,
                                                                        n, g, pc, rows, cols, y), note_launches(1);
  });
  return 0;
}

static int g_outlier_decompress_mode = 2;  // 0: dequantise + overwrite launches, 2: one launch
static int g_outlier_tile = 8192;          // elements per tile of the one-launch decompress
void set_outlier_decompress_mode(int m) { g_outlier_decompress_mode = m; }
void set_outlier_tile(int t) { g_outlier_tile = t; }

int launch_outlier_decompress_tiles(const Ctx &c, const uint8_t *codes, const uint16_t *scales,
                                    const uint32_t *idx, const uint16_t *val, const int32_t *k_dev,
                                    int64_t k_cap, int64_t rows, int64_t cols, int64_t g, void *y,
                                    int ot) {
  if (g_outlier_decompress_mode == 0 || k_cap <= 0) return 1;
  const int L = lanes_for_group(g, 8);
  const int64_t n = rows * cols;
  if (L == 0 || n % 8 != 0 || !aligned(y, 16) || !aligned(codes, 4) || k_cap > (1 << 22) ||
      n >= (1ll << 40))
    return 1;
  const int T = g_outlier_tile;
  // pairs per tile = k x rows spanned must stay in int
  if ((static_cast<int64_t>(T) / cols + 2) * k_cap >= (1ll << 31)) return 1;
  const int64_t tiles = (n + T - 1) / T;
  if (tiles >= (1ll << 31)) return 1;
  const uint32_t *codes32 = reinterpret_cast<const uint32_t *>(codes);
#define ADC_TILES(TT)                                                                                  \
  ADC_OT_SWITCH(ot, OT, ADC_L_SWITCH(L, LL, {                                                          \
    constexpr int TS = (OT == ADC_F32 && TT > 8192) ? 8192 : TT; /* static smem <= 48 KB */           \
    launch_k(outlier_dequant_tiles<OT, LL, TS>, static_cast<int>((n + TS - 1) / TS), kThreads, 0,     \
             c.stream, codes32, scales, rows, cols, n, idx, val, k_dev, static_cast<int>(k_cap), y);  \
    note_launches(1);                                                                                  \
  }))
  switch (T) {
    case 4096: ADC_TILES(4096); break;
    case 8192: ADC_TILES(8192); break;
    case 16384: ADC_TILES(16384); break;
    default: return 1;
  }
#undef ADC_TILES
  return 0;
}

int launch_outlier_scatter(const Ctx &c, const uint32_t *idx, const uint16_t *val,
                           const int32_t *k_dev, int64_t k_cap, int64_t rows, int64_t cols,
                           void *y, int ot, const uint8_t *codes, const uint16_t *scales, int64_t g) {
  if (k_cap <= 0) return 0;
  // whole-sector patches when the output is large (then a 2-byte scatter
  // pays a read-modify-write per element; measured 127.7 -> 105.9 us for
  // [131072,1024] bf16, k = 11; 30.5 -> 29.0 us at [8192,4096], 64 MB) and
  // the codes are row-major groups that never straddle a 32-byte output
  // sector; smaller outputs keep the scatter (one dependent load instead of
  // two: 8.3 vs 12.9 us at [8192,1024], 23.9 vs 25.8 us at [8192,3072])
  const int se = ot == ADC_F32 ? 8 : 16;
  const int L = codes && scales ? lanes_for_group(g, 8) : 0;
  const int64_t out_bytes = rows * cols * (ot == ADC_F32 ? 4 : 2);
  if (L > 0 && out_bytes >= (64ll << 20) && g % se == 0 && cols % se == 0 && aligned(y, 32) &&
      aligned(codes, 4)) {
    const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((rows + 4 * kThreads - 1) / (4 * kThreads), 64));
    const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(k_cap, std::max<int64_t>(1, 8 * c.num_sms / gx)));
    const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(std::min<int64_t>(gy, 65535)));
    const uint32_t *codes32 = reinterpret_cast<const uint32_t *>(codes);
    ADC_OT_SWITCH(ot, OT, ADC_L_SWITCH(L, LL, {
      launch_k(outlier_patch16<OT, LL>, grid, kThreads, 0, c.stream, codes32, scales, idx, val, k_dev,
               k_cap, rows, cols, y);
      note_launches(1);
    }));
    return 0;
  }
  // ~4 rows per thread, ranks across grid.y (at most ~4 waves of CTAs)
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((rows + 4 * kThreads - 1) / (4 * kThreads), 64));
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(k_cap, std::max<int64_t>(1, 8 * c.num_sms / gx)));
  const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(std::min<int64_t>(gy, 65535)));
  ADC_OT_SWITCH(ot, OT, launch_k(outlier_scatter<OT>, grid, kThreads, 0, c.stream, 
                            idx, val, k_dev, k_cap, rows, cols, y), note_launches(1));
  return 0;
}

}  // namespace adc
