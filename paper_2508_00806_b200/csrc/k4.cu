// K4 in ONE pass: the outlier-separated compressor (codec.py:308-341) as a
// persistent cooperative kernel, one 512-thread CTA per SM, the input read
// from HBM once.
//
// Tiling.  The grid is strips x slabs: a CTA owns the rows [r0, r1) of one
// column strip of at most 1024 columns (whole 128-groups).  Its tile reaches
// shared memory through the TMA engine in 16 KB chunks of whole tile rows
// (cp.async.bulk, one mbarrier per slot).  If the tile fits, every chunk stays
// resident; otherwise the chunks stream through a ring of slots.
//
// Thread (p, u) owns the 16 columns [16u, 16u + 16) of the strip in the rows
// p, p + P, ... (P = 512 / (W / 16) row lanes).  A 128-group is 8 lanes.  For
// every row it holds, from two conflict-free 16-byte shared loads:
//   A1. column |x| sums: |h| as f32 (shared with the quotients below) ->
//       float64 (F2F) -> one DADD into 16 per-thread accumulators;
//   A2. the group's symmetric codes with the PREDICTED channel set zeroed
//       (the previous call's flags, kept in the workspace; zero-filled = "no
//       outliers"): group abs-max over 8 lanes, scale, Markstein-rounded
//       quotients two per FFMA2, saturating nibble pack, 8-byte code store.
// B.  The P row lanes are folded through shared memory and the strip's column
//     partials go to a global float64 accumulator with ONE bulk reduction
//     (cp.reduce.async.bulk .add.f64, in L2); grid barrier = one release-add
//     per CTA on a monotonic counter + acquire polls.
// C.  Every CTA reads the column totals and evaluates mean / std / z / flags /
//     ranks itself (numpy's pairwise tree, host-built), no finisher CTA.
// D.  Groups whose channel set differs from the prediction are re-quantised
//     (from shared memory when resident, else from global memory).  When the
//     prediction holds -- steady state: outlier channels persist (PAPER.md
//     Fig. 4a) -- D does nothing and x was read exactly once.
// E.  The float16 values of the flagged channels go to the (k, rows) side
//     buffer (codec.py:339-340).
//
// Exactness: f16 values are integer multiples of
// 2^-24 below 2^16, so every float64 partial sum -- thread, fold, bulk
// reduction -- is exact (hence order-free) while a column total is below
// 2^29.  A finite total >= 2^29
// makes every CTA recompute its share of the columns in numpy's row order
// (slow, exact) behind a second barrier.  Non-finite elements (f16 overflow,
// inf, NaN) are caught by the group abs-max (A2/D), by the side-buffer
// gather (A/E) and by non-finite column totals.  bf16: |x| in [2^-17, 65536)
// is exactly representable in f16, so such values ARE f16(x); a 16-element
// unit holding a smaller value converts each element (numpy's
// astype(float16)).
//
// Eligibility (host side): g = 128, cols % 128 == 0, cols <= 16384, bf16 or
// f16 input, 16-byte aligned buffers, n < 2^31.  Otherwise the caller uses
// the two-launch path (colreduce + group_quant_fast), identical bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <functional>
#include <vector>

#include "common.cuh"
#include "launch.h"
#include "quant.cuh"

namespace adc {

constexpr int kOT = 512;  // threads per CTA
constexpr int kOW = kOT / 32;
constexpr int kOMaxSlots = 16;
constexpr int kOMaxLeaves = 128;  // cols <= 16384
constexpr int kOStripCols = 1024;
constexpr double kOExact = 536870912.0;  // 2^29

// numpy's pairwise_sum_DOUBLE tree for n = cols (block 128, unroll 8, split
// n/2 - (n/2) % 8), flattened on the host: leaves left to right, internal
// nodes ordered by height (node ids: leaves 0..nl-1, internal nl + j).
struct OTree {
  int n_leaves, n_levels;
  int16_t leaf_lo[kOMaxLeaves];
  uint8_t leaf_n[kOMaxLeaves];  // 1..128
  uint8_t left[kOMaxLeaves], right[kOMaxLeaves];
  uint8_t level_end[16];  // internal nodes of height <= h + 1: [0, level_end[h])
};

static bool build_tree(int n, OTree &t) {
  struct Internal { int l, r, h; };
  std::vector<Internal> in;
  std::vector<std::pair<int, int>> leaves;
  std::function<std::pair<int, int>(int, int)> rec = [&](int lo, int m) -> std::pair<int, int> {
    if (m <= 128) {
      leaves.emplace_back(lo, m);
      return {static_cast<int>(leaves.size()) - 1, 0};
    }
    const int h = m / 2 - (m / 2) % 8;
    const auto a = rec(lo, h), b = rec(lo + h, m - h);
    in.push_back({a.first, b.first, 1 + std::max(a.second, b.second)});
    return {-static_cast<int>(in.size()), in.back().h};
  };
  rec(0, n);
  const int nl = static_cast<int>(leaves.size()), ni = static_cast<int>(in.size());
  if (nl > kOMaxLeaves || nl + ni > 255) return false;
  std::vector<int> order(ni), pos(ni);
  for (int i = 0; i < ni; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return in[x].h < in[y].h; });
  for (int i = 0; i < ni; ++i) pos[order[i]] = i;
  auto id = [&](int enc) { return enc >= 0 ? enc : nl + pos[-enc - 1]; };
  t = OTree{};
  t.n_leaves = nl;
  for (int i = 0; i < nl; ++i) {
    t.leaf_lo[i] = static_cast<int16_t>(leaves[i].first);
    t.leaf_n[i] = static_cast<uint8_t>(leaves[i].second);
  }
  int levels = 0;
  for (int j = 0; j < ni; ++j) {
    const Internal &v = in[order[j]];
    t.left[j] = static_cast<uint8_t>(id(v.l));
    t.right[j] = static_cast<uint8_t>(id(v.r));
    levels = std::max(levels, v.h);
    t.level_end[v.h - 1] = static_cast<uint8_t>(j + 1);
  }
  t.n_levels = levels;
  return levels <= 16;
}

struct OArgs {
  const uint16_t *x;
  int64_t rows, cols;
  int strips, slabs;  // grid = strips * slabs
  int rbase, rrem;    // slab i holds rbase + (i < rrem) rows
  int chunk_rows;     // rows per chunk (one chunk = chunk_rows * strip width * 2 bytes <= slot_bytes)
  int n_slots;        // shared slots; a CTA whose chunks all fit keeps them resident
  int slot_bytes;
  int stats_off;      // byte offset of the statistics area (0: overlays the slots, streamed tiles)
  int pred_off;       // byte offset of the predicted flags (cols + 16 bytes, never overlaid)
  double thr;
  int64_t k_cap;
  double *sacc;     // [2][cols] scaled float64 column accumulators (double-buffered, zero at rest)
  double *sseq;     // [cols] numpy row-order sums (only when some total >= 2^29)
  uint32_t *ctl;    // [0] barrier arrivals (monotonic), [1] their base for the next call,
                    // [2] epoch (accumulator parity), [3] cols of the last call
  uint8_t *pflag;   // [cols] previous call's flags (the prediction)
  uint8_t *codes;
  uint16_t *scales;
  uint32_t *idx;
  uint16_t *val;
  int32_t *k_out;
  uint32_t *err;
  int trace;
  int dbg;        // timing experiments only (adc_set_option("k4_dbg")): 1 exit after A (results invalid)
  OTree tree;
};

// Phase timestamps of the last traced launch (tuning): per CTA, [0]
// globaltimer at entry, then clock64 deltas at phase ends.
constexpr int kOTraceSlots = 64;  // [0..15] CTA phases (thread 0), [32+w] / [48+w] warp w entry / exit
constexpr int kOTraceCtas = 1024;
__device__ unsigned long long g_k4trace[kOTraceCtas * kOTraceSlots];
#define K4TRACE(slot)                                                                            \
  do {                                                                                           \
    if (a.trace && tid == 0 && b < kOTraceCtas)                                                  \
      g_k4trace[b * kOTraceSlots + (slot)] = static_cast<unsigned long long>(clock64() - t_0); \
  } while (0)

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_arrive(uint32_t *cnt) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
}
__device__ __forceinline__ void grid_wait(const uint32_t *cnt, uint32_t target) {
  while (static_cast<int32_t>(ld_acquire_u32(cnt) - target) < 0) {
  }
}
// thread 0 arrives and waits; the CTA synchronises around it
__device__ __forceinline__ void cta_grid_sync(uint32_t *cnt, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    grid_arrive(cnt);
    grid_wait(cnt, target);
  }
  __syncthreads();
}

// Rare quantiser cases (kept out of line: the hot loop must stay small for
// the instruction cache): a subnormal or zero scale, or a bf16 group whose
// maximum is so small that the f16 rounding of its elements matters.
template <bool BF>
__device__ __noinline__ uint2 quant16_slow(uint4 a, uint4 c, uint32_t s_bits, bool native) {
  using R = Raw<BF ? ADC_BF16 : ADC_F16>;
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
  uint32_t t[16];
  if (!BF || native) {
    const float s0 = h2f(s_bits), sc = s0 == 0.f ? 1.f : s0, inv = rcp_approx(sc);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      t[2 * i] = sym_tbits_clip2(R::lo(w[i]), sc, inv);
      t[2 * i + 1] = sym_tbits_clip2(R::hi(w[i]), sc, inv);
    }
  } else {
    unit_codes_exact<BF, 8>(w, h2f(s_bits), 0.f, false, t);
  }
  return make_uint2(pack8_tbits_sat(t), pack8_tbits_sat(t + 8));
}

// Symmetric codes of a lane's 16 elements (raw words in load order; the
// abs-max runs over ab = |w| & channel mask), the 128-group spread over 8
// aligned lanes.  Every lane of the warp calls (lanes without data pass
// zeros).  Codes of zeroed channels are not forced to 0 here (the caller ANDs
// the code words): the abs-max alone decides the scale.
template <bool BF>
__device__ __forceinline__ uint2 quant16(const uint32_t *w, const uint32_t *ab, uint16_t &s_bits, bool &bad) {
  using R = Raw<BF ? ADC_BF16 : ADC_F16>;
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) m = __vmaxu2(m, ab[i]);
  m = __vmaxu2(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = __vmaxu2(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = __vmaxu2(m, __shfl_xor_sync(0xffffffffu, m, 4));
  const uint32_t top = max(m & 0xffffu, m >> 16);
  // fast: 2^-11 <= top < 65536 (bf16: the value IS f16(top); f16: finite):
  // s = f16(top / 8) is a normal f16 (top / 8 is exact in f32)
  const bool fast = BF ? (top - 0x3a00u < 0x4780u - 0x3a00u) : (top - 0x1000u < 0x7c00u - 0x1000u);
  if (!fast) {
    bool native = true;
    if (BF) {
      bad = top >= 0x4780u;     // >= 65536 rounds to f16 inf (also inf / NaN)
      native = top >= 0x3900u;  // top >= 2^-13: tiny-value rounding is code-neutral
      s_bits = sym_scale_bits(bf16_bits_to_f16_bits(top));
    } else {
      bad = top >= 0x7c00u;
      s_bits = sym_scale_bits(top);
    }
    return quant16_slow<BF>(make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]), s_bits, native);
  }
  bad = false;
  const float topf = BF ? __uint_as_float(top << 16) : h2f(top);
  s_bits = __half_as_ushort(__float2half_rn(topf * 0.125f));
  // correctly rounded h/s two lanes per FMUL2 / FFMA2 (Markstein), RNE by the
  // magic add, the clips in the saturating pack
  const float sc = h2f(s_bits), inv = rcp_approx(sc);
  const uint64_t inv2 = f2_pack(inv, inv), ns2 = f2_pack(-sc, -sc), mg2 = f2_pack(kMagic8, kMagic8);
  uint32_t t[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t h2 = f2_pack(R::lo(w[i]), R::hi(w[i]));
    const uint64_t r0 = f2_mul(h2, inv2);
    const uint64_t r1 = f2_fma(f2_fma(r0, ns2, h2), inv2, r0);
    float tl, th;
    f2_unpack(f2_add(r1, mg2), tl, th);
    t[2 * i] = __float_as_uint(tl);
    t[2 * i + 1] = __float_as_uint(th);
  }
  return make_uint2(pack8_tbits_sat(t), pack8_tbits_sat(t + 8));
}

// quant16 on precomputed f32 values of the unit (f[2i] / f[2i+1] = low /
// high element of word i) and the lane's abs-max word mx.
template <bool BF>
__device__ __forceinline__ uint2 quant16f(const uint32_t *w, const float *f, uint32_t mx, uint16_t &s_bits,
                                          bool &bad) {
  uint32_t m = mx;
  m = __vmaxu2(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = __vmaxu2(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = __vmaxu2(m, __shfl_xor_sync(0xffffffffu, m, 4));
  const uint32_t top = max(m & 0xffffu, m >> 16);
  const bool fast = BF ? (top - 0x3a00u < 0x4780u - 0x3a00u) : (top - 0x1000u < 0x7c00u - 0x1000u);
  if (!fast) {
    bool native = true;
    if (BF) {
      bad = top >= 0x4780u;
      native = top >= 0x3900u;
      s_bits = sym_scale_bits(bf16_bits_to_f16_bits(top));
    } else {
      bad = top >= 0x7c00u;
      s_bits = sym_scale_bits(top);
    }
    return quant16_slow<BF>(make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]), s_bits, native);
  }
  bad = false;
  const float topf = BF ? __uint_as_float(top << 16) : h2f(top);
  s_bits = __half_as_ushort(__float2half_rn(topf * 0.125f));
  const float sc = h2f(s_bits), inv = rcp_approx(sc);
  const uint64_t inv2 = f2_pack(inv, inv), ns2 = f2_pack(-sc, -sc), mg2 = f2_pack(kMagic8, kMagic8);
  uint32_t t[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t h2 = f2_pack(f[2 * i], f[2 * i + 1]);
    const uint64_t r0 = f2_mul(h2, inv2);
    const uint64_t r1 = f2_fma(f2_fma(r0, ns2, h2), inv2, r0);
    float tl, th;
    f2_unpack(f2_add(r1, mg2), tl, th);
    t[2 * i] = __float_as_uint(tl);
    t[2 * i + 1] = __float_as_uint(th);
  }
  return make_uint2(pack8_tbits_sat(t), pack8_tbits_sat(t + 8));
}

// Zero masks of 16 columns (8 words) from 16 flag bytes (0/1), in load order
// (the half at +8*sw first).
__device__ __forceinline__ void masks16(const uint8_t *flag16, int sw, uint32_t *mk) {
  const uint4 f = *reinterpret_cast<const uint4 *>(flag16);
  const uint2 h0 = sw ? make_uint2(f.z, f.w) : make_uint2(f.x, f.y);
  const uint2 h1 = sw ? make_uint2(f.x, f.y) : make_uint2(f.z, f.w);
#pragma unroll
  for (int i = 0; i < 8; ++i) mk[i] = 0xffffffffu;
  zero_apply8(mk, h0);
  zero_apply8(mk + 4, h1);
}

// Code-word nibble masks of the 8 zero masks (0xF where the channel is kept).
__device__ __forceinline__ uint2 nibble_masks(const uint32_t *mk) {
  uint32_t c[2] = {0u, 0u};
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if ((mk[j >> 1] >> (16 * (j & 1))) & 1u) c[j >> 3] |= 0xfu << (4 * (j & 7));
  return make_uint2(c[0], c[1]);
}

// One row-unit: optional column sums, quantise with mask mk, store the codes
// (in column order) and the group's scale.  Every lane of the warp calls; act
// = this lane holds a row (a group's 8 lanes agree).
struct Unit {
  int sw;
  bool leader;  // lane 0 of the 8-lane group
};
// outputs of the quantiser (passed by value to out-of-line helpers: a
// reference to the kernel's parameter block would copy it to local memory)
struct QOut {
  uint8_t *codes;
  uint16_t *scales;
  uint32_t *err;
};

// Column sums of one unit on the slow path (a zero, a tiny bf16 value, or a
// predicted-outlier lane): h = f16(x) -> f32 -> float64, exactly numpy's
// astype(float16) then float64.
template <bool BF>
__device__ __forceinline__ void colsum16_slow(double *acc, uint4 v0, uint4 v1) {
  const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t h = (BF ? bf2_to_h2(w[i]) : w[i]) & 0x7fff7fffu;
    acc[2 * i] = __dadd_rn(acc[2 * i], static_cast<double>(lo_f(h)));
    acc[2 * i + 1] = __dadd_rn(acc[2 * i + 1], static_cast<double>(hi_f(h)));
  }
}

// One row-unit (16 elements of a row in load order): column |h| sums (SUM)
// and the group's symmetric codes with the zero mask mk; stores the codes
// (column order) and the group's scale.  Every lane of the warp calls; act =
// this lane holds a row (a group's 8 lanes agree).
//   sums: bf16 values in [2^-17, 65536) ARE their f16 rounding, so |x| as
//   f32 -> float64 (F2F) is exact; f16 values always convert exactly.  The
//   same f32 values feed the quotients.
template <bool BF, bool SUM, bool QUANT = true>
__device__ __forceinline__ void row_unit(const Unit &U, bool act, uint4 v0, uint4 v1, const uint32_t *mk, uint2 cm,
                                         double *acc, uint2 *code_dst, uint16_t *scale_dst, uint32_t *err) {
  using R = Raw<BF ? ADC_BF16 : ADC_F16>;
  const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  uint32_t mx = 0, mn = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mx = __vmaxu2(mx, w[i] & mk[i] & 0x7fff7fffu);                  // abs-max of the kept channels
    if (SUM && BF) mn = __vminu2(mn, w[i] & 0x7fff7fffu);            // abs-min of all channels
  }
  float f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[2 * i] = R::lo(w[i]);
    f[2 * i + 1] = R::hi(w[i]);
  }
  if (SUM && act) {
    // bf16: a unit holding a zero or a value below 2^-17 (any channel) takes
    // the converting path
    if (!BF || min(mn & 0xffffu, mn >> 16) >= 0x3700u) {
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = __dadd_rn(acc[j], static_cast<double>(fabsf(f[j])));
    } else {
      colsum16_slow<BF>(acc, v0, v1);
    }
  }
  if (!QUANT) return;
  uint16_t s_bits;
  bool bad;
  uint2 cw = quant16f<BF>(w, f, mx, s_bits, bad);
  if (!act) return;
  cw.x &= cm.x;
  cw.y &= cm.y;
  *code_dst = U.sw ? make_uint2(cw.y, cw.x) : cw;
  if (U.leader) {
    *scale_dst = s_bits;
    if (bad) raise_err(err, ADC_ERR_NONFINITE);
  }
}

// A, the flagged-channel side buffer under the prediction: one warp copies
// the predicted outlier columns of a resident chunk (cr rows) from shared
// memory to val[rank][row] (codec.py:339-340).  Consecutive lanes take
// consecutive rows of one column, so every store instruction writes whole
// 32-byte sectors.
template <bool BF>
__device__ __noinline__ void capture_chunk(const unsigned char *chunk, int rowb, int cr, int tc0, const uint16_t *ptcol,
                                           int ntp, int rank0, int64_t row0, int64_t rows, int64_t k_cap, uint16_t *val,
                                           uint32_t *err) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  for (int it = lane; it < ntp * cr; it += 32) {
    const int j = it / cr, r = it - j * cr;
    const int rank = rank0 + j;
    const uint32_t v = *reinterpret_cast<const uint16_t *>(chunk + r * rowb + (ptcol[j] - tc0) * 2);
    const uint32_t h = BF ? bf16_bits_to_f16_bits(v) : v;
    bad |= (h & 0x7fffu) >= 0x7c00u;
    if (rank < k_cap) val[static_cast<int64_t>(rank) * rows + row0 + r] = static_cast<uint16_t>(h);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_err(err, ADC_ERR_NONFINITE);
}

// D, out of line: re-quantise the lane's unit in every row of the tile with
// the actual channel set (from shared memory when resident, else global).
template <bool BF>
__device__ __noinline__ void redo_rows(QOut q, const uint16_t *x, int64_t cols, int CR, int slot_bytes, Unit U,
                                       bool redo, uint4 mk0, uint4 mk1, const unsigned char *slots, bool resident,
                                       int64_t r0, int nrows, int W, int p, int P, int u, int tc0) {
  const uint32_t mk[8] = {mk0.x, mk0.y, mk0.z, mk0.w, mk1.x, mk1.y, mk1.z, mk1.w};
  const uint2 cm = nibble_masks(mk);
#pragma unroll 1
  for (int base = 0; base < nrows; base += P) {  // warp-uniform trip count
    const int rr = base + p;
    const bool act = redo && rr < nrows;
    const int64_t e = (r0 + rr) * cols + tc0 + 16 * u;
    uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
    if (!act) {
    } else if (resident) {
      const int c = rr / CR;
      const unsigned char *src = slots + c * slot_bytes + (rr - c * CR) * W * 2 + 32 * u;
      v0 = *reinterpret_cast<const uint4 *>(src + 16 * U.sw);
      v1 = *reinterpret_cast<const uint4 *>(src + 16 * (1 - U.sw));
    } else {
      const uint4 *src = reinterpret_cast<const uint4 *>(x + e);
      v0 = __ldcg(src + U.sw);
      v1 = __ldcg(src + 1 - U.sw);
    }
    row_unit<BF, false>(U, act, v0, v1, mk, cm, nullptr, reinterpret_cast<uint2 *>(q.codes + e / 2),
                        q.scales + (e >> 7), q.err);
  }
}

// numpy pairwise sum over the S[] terms (squared deviations when `mean` is
// given): leaves by 8-lane groups (the 8 interleaved accumulators of a
// 128-block), internal nodes level by level by warp 0.  Every thread calls;
// all receive 0.0 + sum.
__device__ __noinline__ double tree_sum(const OTree &tr, const double *S, bool squared, double mean, double *s_tv,
                                        double *s_out) {
  const int tid = threadIdx.x, lane = tid & 31, j8 = tid & 7;
  constexpr int ng = kOT / 8;
  for (int g0 = 0; g0 < tr.n_leaves; g0 += ng) {
    const int g = g0 + (tid >> 3);
    const bool valid = g < tr.n_leaves;
    const int lo = valid ? tr.leaf_lo[g] : 0, m = valid ? tr.leaf_n[g] : 0;
    const int stop = m - (m % 8);
    double r = 0.0;
    if (valid && m >= 8) {
      for (int i = j8; i < stop; i += 8) {
        double v = S[lo + i];
        if (squared) {
          const double d = __dsub_rn(v, mean);
          v = __dmul_rn(d, d);
        }
        r = i == j8 ? v : __dadd_rn(r, v);
      }
    }
    // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
    const double x1 = __dadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1, 8));
    const double x2 = __dadd_rn(x1, __shfl_down_sync(0xffffffffu, x1, 2, 8));
    double x3 = __dadd_rn(x2, __shfl_down_sync(0xffffffffu, x2, 4, 8));
    if (valid && j8 == 0) {
      if (m < 8) x3 = 0.0;
      for (int i = stop; i < m; ++i) {
        double v = S[lo + i];
        if (squared) {
          const double d = __dsub_rn(v, mean);
          v = __dmul_rn(d, d);
        }
        x3 = __dadd_rn(x3, v);
      }
      s_tv[g] = x3;
    }
  }
  __syncthreads();
  if (tid < 32) {
    const int nl = tr.n_leaves;
    int beg = 0;
    for (int h = 0; h < tr.n_levels; ++h) {
      const int end = tr.level_end[h];
      for (int q = beg + lane; q < end; q += 32) s_tv[nl + q] = __dadd_rn(s_tv[tr.left[q]], s_tv[tr.right[q]]);
      __syncwarp();
      beg = end;
    }
    if (lane == 0) *s_out = __dadd_rn(0.0, s_tv[beg == 0 ? 0 : nl + beg - 1]);
  }
  __syncthreads();
  return *s_out;
}

// numpy row-order column sums (only when some column total reaches 2^29):
// the columns shared out over the grid, one thread per column.
template <bool BF>
__device__ __noinline__ void numpy_order_sums(const uint16_t *x, int64_t rows, int64_t cols, double *out) {
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * kOT + threadIdx.x; c < cols;
       c += static_cast<int64_t>(gridDim.x) * kOT) {
    double sum = 0.0;
#pragma unroll 1
    for (int64_t r = 0; r < rows; ++r) {
      const uint32_t v = x[r * cols + c];
      const uint32_t h = BF ? bf16_bits_to_f16_bits(v) : v;
      sum = __dadd_rn(sum, fabs(static_cast<double>(h2f(h))));
    }
    __stcg(out + c, sum);
  }
}

// E: the flagged channels of the tile, rows [r0, r0 + nrows): val[rank][r] = f16(x[r, col]).
template <bool BF>
__device__ __noinline__ void side_buffer(const uint16_t *x, int64_t rows, int64_t cols, int CR, int slot_bytes,
                                         int64_t k_cap, uint16_t *val, uint32_t *err, const unsigned char *slots,
                                         bool resident, int64_t r0, int nrows, int W, int tc0, const uint16_t *s_tcol,
                                         int nt, int rank0) {
  const int items = nt * nrows;
#pragma unroll 1
  for (int it = threadIdx.x; it < items; it += kOT) {
    const int j = it / nrows, rr = it - j * nrows;
    const int rank = rank0 + j;
    const int cc = s_tcol[j];
    uint32_t v;
    if (resident) {
      const int c = rr / CR;
      v = *reinterpret_cast<const uint16_t *>(slots + c * slot_bytes + (rr - c * CR) * W * 2 + (cc - tc0) * 2);
    } else {
      v = __ldcg(x + (r0 + rr) * cols + cc);
    }
    const uint32_t h = BF ? bf16_bits_to_f16_bits(v) : v;
    if ((h & 0x7fffu) >= 0x7c00u) raise_err(err, ADC_ERR_NONFINITE);
    if (rank < k_cap) val[static_cast<int64_t>(rank) * rows + r0 + rr] = static_cast<uint16_t>(h);
  }
}

template <bool BF>
__global__ void __launch_bounds__(kOT, 1) outlier_onepass(OArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_full[kOMaxSlots];
  __shared__ uint32_t s_done[kOMaxSlots];
  __shared__ __align__(8) uint64_t s_pbar;  // the prediction's copy
  __shared__ double s_red[kOW];
  __shared__ double s_tv[2 * kOMaxLeaves];
  __shared__ double s_stat;
  __shared__ int s_cnt[kOW + 2];
  __shared__ int s_lt[kOW], s_lt1[kOW];
  __shared__ uint32_t s_ctl[3];
  __shared__ uint16_t s_tcol[kOStripCols];  // flagged columns of this strip, ascending
  __shared__ OTree s_tree;
  __shared__ uint16_t s_urank[kOMaxLeaves * 8 + 1];  // predicted flags before each 16-column unit (+ total)
  __shared__ uint16_t s_ptcol[kOStripCols];           // predicted outlier columns of the strip, ascending
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t C = gridDim.x;
  const int b = blockIdx.x;
  const long long t_0 = clock64();
  if (a.trace && lane == 0 && b < kOTraceCtas) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    if (tid == 0) g_k4trace[b * kOTraceSlots] = gt;
    g_k4trace[b * kOTraceSlots + 32 + wid] = gt;
  }
  const int64_t rows = a.rows, cols = a.cols;
  // this CTA's tile: strip columns [tc0, tc0 + W), slab rows [r0, r1)
  const int strip = b % a.strips, slab = b / a.strips;
  const int G = static_cast<int>(cols >> 7);
  const int g0 = G * strip / a.strips, g1 = G * (strip + 1) / a.strips;
  const int tc0 = 128 * g0, W = 128 * (g1 - g0);
  const int64_t r0 = static_cast<int64_t>(slab) * a.rbase + min(slab, a.rrem);
  const int nrows = a.rbase + (slab < a.rrem ? 1 : 0);
  const int CR = a.chunk_rows;
  const int nchunks = (nrows + CR - 1) / CR;
  const bool resident = nchunks <= a.n_slots;
  unsigned char *slots = smem;
  double *S = reinterpret_cast<double *>(smem + a.stats_off);  // [cols]
  uint8_t *s_flag = reinterpret_cast<uint8_t *>(S + cols);     // [cols + 16]
  uint8_t *s_pred = smem + a.pred_off;                          // [cols + 16] previous call's flags

  const int rowb = W * 2;
  auto issue = [&](int c) {  // warp-cooperative: lane i copies rows i, i + 32, ... of chunk c
    const int s = c % a.n_slots;
    const int cr = min(CR, nrows - c * CR);
    if (lane == 0) mbar_expect_tx(&s_full[s], static_cast<uint32_t>(cr * rowb));
    __syncwarp();
    unsigned char *dst = slots + s * a.slot_bytes;
    const uint16_t *src = a.x + (r0 + static_cast<int64_t>(c) * CR) * cols + tc0;
    if (W == cols) {  // contiguous rows: one copy
      if (lane == 0) bulk_g2s(dst, src, static_cast<uint32_t>(cr * rowb), &s_full[s]);
    } else {
      for (int i = lane; i < cr; i += 32) bulk_g2s(dst + i * rowb, src + i * cols, static_cast<uint32_t>(rowb), &s_full[s]);
    }
  };
  if (wid == 0) {  // barriers, then every copy: the prediction first, the chunks behind it
    if (lane == 0) {
#pragma unroll 1
      for (int s = 0; s < a.n_slots; ++s) {
        mbar_init(&s_full[s], 1);
        s_done[s] = 0;
      }
      mbar_init(&s_pbar, 1);
      fence_barrier_init();
      const uint32_t pbytes = static_cast<uint32_t>((cols + 15) & ~15ll);
      mbar_expect_tx(&s_pbar, pbytes);
      bulk_g2s(s_pred, a.pflag, pbytes, &s_pbar);
    }
    __syncwarp();
    K4TRACE(14);
    for (int c = 0; c < min(nchunks, a.n_slots); ++c) issue(c);
    K4TRACE(15);
  } else if (tid == 32) {
    s_ctl[0] = a.ctl[1];  // barrier base
    s_ctl[1] = a.ctl[2];  // epoch
    s_ctl[2] = a.ctl[3];  // cols of the last call (accumulator layout)
  } else if (wid == 2) {  // the pairwise tree, for the statistics
    const uint32_t *src = reinterpret_cast<const uint32_t *>(&a.tree);
    uint32_t *dst = reinterpret_cast<uint32_t *>(&s_tree);
    for (int i = lane; i < static_cast<int>(sizeof(OTree) / 4); i += 32) dst[i] = src[i];
  }
  __syncthreads();  // barrier initialisation visible to every warp
  // the prediction (previous call's flags, in shared memory): exclusive counts per 16-column unit
  {
    const int gu = static_cast<int>(cols / 16);
    int cnt0 = 0, cnt1 = 0;
    mbar_wait(&s_pbar, 0);
    if (2 * tid < gu) {
      const uint4 f = *reinterpret_cast<const uint4 *>(s_pred + 32 * tid);
      cnt0 = __popc(f.x) + __popc(f.y) + __popc(f.z) + __popc(f.w);  // bytes are 0 / 1
    }
    if (2 * tid + 1 < gu) {
      const uint4 f = *reinterpret_cast<const uint4 *>(s_pred + 32 * tid + 16);
      cnt1 = __popc(f.x) + __popc(f.y) + __popc(f.z) + __popc(f.w);
    }
    const int mine = cnt0 + cnt1;
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_cnt[wid] = incl;
    __syncthreads();
    int before = 0;
#pragma unroll
    for (int w2 = 0; w2 < kOW; ++w2) before += w2 < wid ? s_cnt[w2] : 0;
    const int excl = before + incl - mine;
    if (tid == kOT - 1) s_urank[gu] = static_cast<uint16_t>(excl + mine);  // (gu <= 1024 = 2 * kOT)
    if (2 * tid < gu) s_urank[2 * tid] = static_cast<uint16_t>(excl);
    if (2 * tid + 1 < gu) s_urank[2 * tid + 1] = static_cast<uint16_t>(excl + cnt0);
    __syncthreads();
  K4TRACE(18);
  }
  const QOut qo{a.codes, a.scales, a.err};
  // lane mapping: thread (p, u), u = unit of 16 columns of the strip
  const int units = W / 16;
  const int P = kOT / units;
  const int p = tid / units, u = tid - p * units;
  const bool on = p < P;
  Unit U;
  U.sw = (u >> 2) & 1;  // 16-byte halves swapped on lanes 4..7 mod 8: conflict-free LDS.128
  U.leader = (u & 7) == 0;
  uint32_t pmk[8];  // predicted zero masks (previous call's flags), load order
  uint32_t predm = 0;  // predicted outlier columns of the lane (bit j = column 16u + j)
  int prank = 0;       // predicted rank of the first of them
  if (on) {
    masks16(s_pred + tc0 + 16 * u, U.sw, pmk);
#pragma unroll
    for (int j = 0; j < 16; ++j) predm |= static_cast<uint32_t>(s_pred[tc0 + 16 * u + j]) << j;
    prank = s_urank[tc0 / 16 + u];
    if (p == 0)  // the strip's predicted columns, for the chunk captures
      for (uint32_t m = predm; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        s_ptcol[prank - s_urank[tc0 / 16] + __popc(predm & ((1u << j) - 1u))] = static_cast<uint16_t>(tc0 + 16 * u + j);
      }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) pmk[i] = 0xffffffffu;
  }
  K4TRACE(16);
  const uint2 pcm = nibble_masks(pmk);
  __syncthreads();  // s_ptcol
  const int ptc0 = s_urank[tc0 / 16];
  const int ntp = s_urank[(tc0 + W) / 16] - ptc0;  // predicted outlier columns in the strip
  K4TRACE(9);

  // ---- A: column sums + quantisation with the predicted channel set ---------
  double acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0.0;
  {
    // per-thread constants of the row walk: shared source offset (unit u, its
    // swap), code / scale destinations of row p of chunk 0, strides per P rows
    const int sm_off = p * rowb + 32 * u;
    const int64_t e_first = (r0 + p) * cols + tc0 + 16 * u;
    uint2 *cdst0 = reinterpret_cast<uint2 *>(a.codes) + e_first / 16;
    uint16_t *sdst0 = a.scales + (e_first >> 7);
    const int64_t cstep = static_cast<int64_t>(P) * cols / 16, sstep = static_cast<int64_t>(P) * cols / 128;
    const int64_t cchunk = static_cast<int64_t>(CR) * cols / 16, schunk = static_cast<int64_t>(CR) * cols / 128;
    int s = 0;
    uint32_t phase = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int cr = min(CR, nrows - c * CR);
      mbar_wait(&s_full[s], phase);
      if (wid == (c & (kOW - 1)) && ntp > 0 && a.val)
        capture_chunk<BF>(slots + s * a.slot_bytes, rowb, cr, tc0, s_ptcol, ntp, ptc0,
                          r0 + static_cast<int64_t>(c) * CR, rows, a.k_cap, a.val, a.err);
      const unsigned char *src = slots + s * a.slot_bytes + sm_off;
      uint2 *cdst = cdst0;
      uint16_t *sdst = sdst0;
      for (int rr = p; rr - p < cr; rr += P) {  // warp-uniform trip count
        const bool act = on && rr < cr;
        uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
        if (act) {
          v0 = *reinterpret_cast<const uint4 *>(src + 16 * U.sw);
          v1 = *reinterpret_cast<const uint4 *>(src + 16 * (1 - U.sw));
        }
        row_unit<BF, true>(U, act, v0, v1, pmk, pcm, acc, cdst, sdst, a.err);
        src += P * rowb;
        cdst += cstep;
        sdst += sstep;
      }
      cdst0 += cchunk;
      sdst0 += schunk;
      if (!resident) {  // ring: the last warp done with the slot refills it
        __syncwarp();
        uint32_t d = 0;
        if (lane == 0) d = atomicAdd(&s_done[s], 1u);
        d = __shfl_sync(0xffffffffu, d, 0);
        if (d == kOW - 1) {
          if (lane == 0) s_done[s] = 0;
          if (c + a.n_slots < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(c + a.n_slots);
          }
        }
      }
      if (++s == a.n_slots) {
        s = 0;
        phase ^= 1u;
      }
    }
  }
  K4TRACE(1);
  if (a.dbg == 1) return;

  // ---- B: fold the row lanes, one bulk reduction, barrier arrival ----------
  // stage: row lane p's partial of column 16u + j at T[p * units + u][j], 17
  // doubles per unit (the pad keeps lanes' 128-byte runs on distinct banks);
  // the staging area is the statistics area (streamed tiles: the free ring).
  __syncthreads();
  K4TRACE(17);
  double *T = S;  // P * units * 17 doubles
  if (on) {
    double *t = T + (p * units + u) * 17;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      t[8 * U.sw + j] = acc[j];
      t[8 * (1 - U.sw) + j] = acc[8 + j];
    }
  }
  __syncthreads();
  const uint32_t bar_base = s_ctl[0], epoch = s_ctl[1];
  const bool relayout = s_ctl[2] != static_cast<uint32_t>(cols);
  double *sacc = a.sacc + (epoch & 1u) * cols;
  double *sacc_next = a.sacc + ((epoch + 1u) & 1u) * cols;
  uint32_t n_bar = 0;
  if (relayout) {
    // first call on this workspace layout: zero the accumulator behind an extra barrier
    for (int64_t c = static_cast<int64_t>(b) * kOT + tid; c < cols; c += static_cast<int64_t>(C) * kOT)
      __stcg(sacc + c, 0.0);
    __threadfence();
    ++n_bar;
    cta_grid_sync(a.ctl, bar_base + n_bar * C);
  }
  // the strip's column partials straight into the global accumulator (f64
  // reductions in L2, exact: order-free); no async-proxy hand-off (its fence
  // would wait for every code store of phase A)
#pragma unroll 1
  for (int c = tid; c < W; c += kOT) {
    const double *t = T + (c >> 4) * 17 + (c & 15);
    double v = t[0];
#pragma unroll 4
    for (int q = 1; q < P; ++q) v = __dadd_rn(v, t[q * units * 17]);
    if (nrows > 0) atomicAdd(sacc + tc0 + c, v);
  }
  __syncthreads();
  K4TRACE(2);
  ++n_bar;
  if (tid == 0) grid_arrive(a.ctl);
  K4TRACE(3);
  if (tid == 0) grid_wait(a.ctl, bar_base + n_bar * C);
  __syncthreads();
  K4TRACE(13);

  // ---- C: statistics, redundantly in every CTA ------------------------------
  int big = 0, nonfinite = 0;
#pragma unroll 1
  for (int c = tid; c < cols; c += kOT) {
    const double v = __ldcg(sacc + c);
    big |= (v >= kOExact) && (v <= 65504.0 * static_cast<double>(rows));
    nonfinite |= !(v < 0x1p100);  // an f16 inf / NaN element entered the sum as >= 2^128
    S[c] = v;
  }
  // the other accumulator buffer is the next call's: zero it (this call never reads it)
  for (int64_t c = static_cast<int64_t>(b) * kOT + tid; c < cols; c += static_cast<int64_t>(C) * kOT)
    __stcg(sacc_next + c, 0.0);
  {
    const int both = __syncthreads_or(big | (nonfinite << 1));
    big = both & 1;
    nonfinite = both >> 1;
  }
  if (b == 0 && tid == 0 && nonfinite) raise_err(a.err, ADC_ERR_NONFINITE);
  if (big) {
    // some finite total reached 2^29: numpy's row-order sums behind a second barrier
    numpy_order_sums<BF>(a.x, rows, cols, a.sseq);
    __threadfence();
    ++n_bar;
    cta_grid_sync(a.ctl, bar_base + n_bar * C);
    for (int c = tid; c < cols; c += kOT) S[c] = __ldcg(a.sseq + c);
    __syncthreads();
  }
  if (b == 0 && tid == 0) {
    // every CTA read ctl before its first arrival: publish the next call's base / epoch / layout
    a.ctl[1] = bar_base + n_bar * C;
    a.ctl[2] = epoch + 1u;
    a.ctl[3] = static_cast<uint32_t>(cols);
  }
  K4TRACE(4);
  // 1) mean: any-order total (exact below 2^29), else the tree
  double part = 0.0;
#pragma unroll 1
  for (int c = tid; c < cols; c += kOT) part = __dadd_rn(part, S[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
  if (lane == 0) s_red[wid] = part;
  __syncthreads();
  double total = lane < kOW ? s_red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total = __dadd_rn(total, __shfl_xor_sync(0xffffffffu, total, o));
  if (!(total < kOExact)) total = tree_sum(s_tree, S, false, 0.0, s_tv, &s_stat);
  const double mean = __ddiv_rn(__dadd_rn(0.0, total), static_cast<double>(cols));
  K4TRACE(10);
  // 2) population variance through the tree
  const double var = __ddiv_rn(tree_sum(s_tree, S, true, mean, s_tv, &s_stat), static_cast<double>(cols));
  K4TRACE(11);
  const double sigma = __dsqrt_rn(var);
  K4TRACE(5);

  // 3) flags of a contiguous run of columns per thread, ranks by block scan
  int rank_t0;  // flagged columns before the strip (rank of its first flagged column)
  int nt;       // flagged columns in the strip
  {
    const int run = static_cast<int>((cols + kOT - 1) / kOT);  // <= 32
    const int c0 = static_cast<int>(min(cols, static_cast<int64_t>(run) * tid));
    const int c1 = static_cast<int>(min(cols, static_cast<int64_t>(c0 + run)));
    uint32_t fb = 0;
    if (sigma != 0.0) {
      // z = fl(d / sigma), d = fl(s - mean) (numpy), is monotone in d: decided
      // in the d domain against T = fl(thr * sigma) outside a |T| * 2^-46
      // margin (far beyond the quotient's rounding), the correctly rounded
      // division inside it (stats.cuh, outlier_flags_block)
      const double T = __dmul_rn(a.thr, sigma);
      const double T_m = __dadd_rn(__dmul_rn(fabs(T), 0x1p-46), 0x1p-1000);
      const double T_hi = __dadd_rn(T, T_m), T_lo = __dsub_rn(T, T_m);
#pragma unroll 4
      for (int c = c0; c < c1; ++c) {
        const double d = __dsub_rn(S[c], mean);
        bool f = d > T_hi;
        if (!f && !(d < T_lo)) f = __ddiv_rn(d, sigma) > a.thr;
        fb |= (f ? 1u : 0u) << (c - c0);
      }
    }
    const int mine = __popc(fb);
    // flagged columns of this run before the strip's first / past its last column
    auto before_col = [&](int col) {
      return col <= c0 ? 0 : col >= c1 ? mine : __popc(fb & ((1u << (col - c0)) - 1u));
    };
    int lt0 = before_col(tc0), lt1 = before_col(tc0 + W);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
      lt0 += __shfl_xor_sync(0xffffffffu, lt0, o);
      lt1 += __shfl_xor_sync(0xffffffffu, lt1, o);
    }
    if (lane == 31) s_cnt[wid] = incl;
    if (lane == 0) {
      s_lt[wid] = lt0;
      s_lt1[wid] = lt1;
    }
#pragma unroll 1
    for (int c = c0; c < c1; ++c) s_flag[c] = static_cast<uint8_t>((fb >> (c - c0)) & 1u);
    __syncthreads();
    K4TRACE(19);
    int before = 0, total_k = 0, rank_t1 = 0;
    rank_t0 = 0;
#pragma unroll
    for (int w2 = 0; w2 < kOW; ++w2) {
      const int cw = s_cnt[w2];
      before += w2 < wid ? cw : 0;
      total_k += cw;
      rank_t0 += s_lt[w2];
      rank_t1 += s_lt1[w2];
    }
    nt = rank_t1 - rank_t0;
    int pos = before + incl - mine;
    for (uint32_t m = fb; m; m &= m - 1, ++pos) {
      const int q = c0 + __ffs(m) - 1;
      if (b == 0 && a.idx && pos < a.k_cap) a.idx[pos] = static_cast<uint32_t>(q);
      if (q >= tc0 && q < tc0 + W) s_tcol[pos - rank_t0] = static_cast<uint16_t>(q);
    }
    if (b == 0 && tid == 0) {
      if (a.k_out) *a.k_out = total_k;
      if (2 * static_cast<int64_t>(total_k) > cols) raise_err(a.err, ADC_ERR_TOO_MANY_OUTLIERS);
      if (total_k > a.k_cap) raise_err(a.err, ADC_ERR_K_CAP);
    }
  }
  K4TRACE(20);
  // the new prediction (every CTA read the old one before its arrival)
  if (b == 0)
    for (int c = tid; c < cols; c += kOT) a.pflag[c] = s_flag[c];
  __syncthreads();
  K4TRACE(6);

  // ---- D: re-quantise the groups whose channel set differs from the prediction
  {
    uint32_t amk[8];
    uint32_t dif = 0;
    if (on) {
      masks16(s_flag + tc0 + 16 * u, U.sw, amk);
#pragma unroll
      for (int i = 0; i < 8; ++i) dif |= amk[i] ^ pmk[i];
    }
    // a group is redone when any of its 8 lanes changed
    const uint32_t bal = __ballot_sync(0xffffffffu, dif != 0u);
    const bool redo = on && (bal & (0xffu << (lane & 24))) != 0u;
    if (bal)
      redo_rows<BF>(qo, a.x, cols, CR, a.slot_bytes, U, redo, make_uint4(amk[0], amk[1], amk[2], amk[3]),
                    make_uint4(amk[4], amk[5], amk[6], amk[7]), slots, resident, r0, nrows, W, p, P, u, tc0);
  }
  K4TRACE(7);

  // ---- E: side buffer: val[rank][r] = f16(x[r, idx[rank]]) for the tile,
  // unless the prediction held for every column (then A already wrote it)
  int miss = 0;
#pragma unroll 1
  for (int c = tid; c < cols; c += kOT) miss |= s_flag[c] != s_pred[c];
  miss = __syncthreads_or(miss);
  if (miss && a.val && nt > 0 && nrows > 0)
    side_buffer<BF>(a.x, rows, cols, CR, a.slot_bytes, a.k_cap, a.val, a.err, slots, resident, r0, nrows, W, tc0,
                    s_tcol, nt, rank_t0);
  K4TRACE(8);
  if (a.trace && lane == 0 && b < kOTraceCtas) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    if (tid == 0) g_k4trace[b * kOTraceSlots + 12] = gt;
    g_k4trace[b * kOTraceSlots + 48 + wid] = gt;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int optin_smem() {
  static int v = 0;
  if (!v) {
    int dev = 0, s = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&s, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || s <= 0)
      s = 227 * 1024;
    v = s;
  }
  return v;
}

static std::atomic<int> g_k4_trace{0};
static std::atomic<int> g_k4_dbg{0};
void set_k4_dbg(int v) { g_k4_dbg.store(v, std::memory_order_relaxed); }
// 0: two launches, 1: single pass wherever eligible, 2: automatic (default):
// the single pass where it measured faster -- tall tensors of <= 1024
// columns (one strip), >= 2^25 elements ([131072,1024] bf16: 116 vs 138 us);
// at [8192,1024] / [8192,4096] the two launches win (18.0 vs 22.3 us, 44.8 vs
// 47.5 us: the one-wave cooperative launch, the serial statistics tail and
// the per-row 2-byte work cost more than the L2 re-read they save).
static std::atomic<int> g_k4_mode{-1};

int k4_mode() {
  int v = g_k4_mode.load(std::memory_order_relaxed);
  if (v < 0) {
    const char *e = getenv("ADC_OUTLIER_PATH");
    v = !e ? 2 : e[0] == '0' ? 0 : e[0] == '1' ? 1 : 2;
    g_k4_mode.store(v, std::memory_order_relaxed);
  }
  return v;
}
void set_k4_mode(int v) { g_k4_mode.store(v, std::memory_order_relaxed); }
void set_k4_trace(int v) { g_k4_trace.store(v, std::memory_order_relaxed); }
int read_k4_trace(unsigned long long *host, int n) {
  if (n > kOTraceCtas * kOTraceSlots) n = kOTraceCtas * kOTraceSlots;
  return cudaMemcpyFromSymbol(host, g_k4trace, sizeof(unsigned long long) * n) == cudaSuccess ? n : -1;
}

template <bool BF>
static int onepass_go(const Ctx &c, const OArgs &a, size_t smem, int grid) {
  auto kern = outlier_onepass<BF>;
  static size_t configured = 0;  // per instantiation
  if (smem > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    configured = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kOT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency of the grid barrier
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  note_launches(1);
  return 1;
}

int launch_outlier_k4(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols, int64_t g,
                      double thr, int64_t k_cap, const Workspace &ws, uint8_t *codes,
                      uint16_t *scales, uint32_t *idx, uint16_t *val, int32_t *k_out,
                      uint32_t *err) {
  const int mode = k4_mode();
  if (mode == 0) return 0;
  const int64_t n = rows * cols;
  if (mode == 2 && (cols > kOStripCols || n < (1ll << 25))) return 0;
  if (g != 128 || cols % 128 || cols > 16384 || n >= (1ll << 31)) return 0;
  if (dt != ADC_BF16 && dt != ADC_F16) return 0;
  if (reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(codes) % 16) return 0;
  if (k_cap > 0 && (!idx || !val)) return 0;
  OArgs a{};
  a.x = static_cast<const uint16_t *>(x);
  a.rows = rows;
  a.cols = cols;
  {
    static thread_local int tree_cols = -1;
    static thread_local OTree tree;
    if (tree_cols != static_cast<int>(cols)) {
      if (!build_tree(static_cast<int>(cols), tree)) return 0;
      tree_cols = static_cast<int>(cols);
    }
    a.tree = tree;
  }
  const int G = static_cast<int>(cols / 128);
  a.strips = (G + kOStripCols / 128 - 1) / (kOStripCols / 128);
  a.slabs = static_cast<int>(std::min<int64_t>(c.num_sms / a.strips, rows));
  if (a.slabs < 1) return 0;
  a.rbase = static_cast<int>(rows / a.slabs);
  a.rrem = static_cast<int>(rows % a.slabs);
  const int grid = a.strips * a.slabs;
  const int wmax = 128 * ((G + a.strips - 1) / a.strips);
  // chunk = P_min rows of the widest strip (each row lane one row per chunk), 16 KB
  a.chunk_rows = std::max(1, 16384 / wmax);  // 32 KB: two rows per row lane of the widest strip
  a.slot_bytes = a.chunk_rows * wmax * 2;
  const int64_t slab_rows = a.rbase + (a.rrem ? 1 : 0);
  const int64_t nchunks = (slab_rows + a.chunk_rows - 1) / a.chunk_rows;
  const int static_smem = 8192;  // mbarriers, tree values, strip column list (conservative)
  const int64_t budget = optin_smem() - static_smem;
  // statistics area: S[cols] doubles + flags; during B it stages P * W + W fold doubles
  const int p_max = kOT / (wmax / 16);
  const int64_t stats = std::max<int64_t>(cols * 8 + cols + 16,
                                          (static_cast<int64_t>(p_max) * (wmax / 16) * 17 + wmax) * 8);
  const int64_t stats_al = (stats + 127) / 128 * 128;
  const int64_t pred_al = (cols + 16 + 127) / 128 * 128;
  if (nchunks * a.slot_bytes + stats_al + pred_al <= budget && nchunks <= kOMaxSlots) {
    a.n_slots = static_cast<int>(nchunks);
    a.stats_off = static_cast<int>(nchunks * a.slot_bytes);
  } else {
    a.n_slots = static_cast<int>(std::min<int64_t>(kOMaxSlots, (budget - pred_al) / a.slot_bytes));
    a.stats_off = 0;  // overlays the ring (free once A is done)
    if (a.n_slots < 2 || stats_al + pred_al > budget) return 0;
  }
  a.pred_off = static_cast<int>(std::max<int64_t>(a.stats_off + stats_al, static_cast<int64_t>(a.n_slots) * a.slot_bytes));
  const size_t smem = static_cast<size_t>(a.pred_off + pred_al);
  a.thr = thr;
  a.k_cap = std::max<int64_t>(k_cap, 0);
  a.sacc = ws.k4acc;
  a.sseq = ws.colsum;
  a.ctl = ws.counters + 4;
  a.pflag = ws.pflag;
  a.codes = codes;
  a.scales = scales;
  a.idx = idx;
  a.val = val;
  a.k_out = k_out;
  a.err = err;
  a.trace = g_k4_trace.load(std::memory_order_relaxed);
  a.dbg = g_k4_dbg.load(std::memory_order_relaxed);
  return dt == ADC_BF16 ? onepass_go<true>(c, a, smem, grid) : onepass_go<false>(c, a, smem, grid);
}

}  // namespace adc
