// K3 / K3': per-channel symmetric int4 (scheme_for(QKV_MATRIX), codec.py:76-77).
//
// Reference semantics: group c = column c over all rows (_grouped_view with
// PER_CHANNEL, codec.py:181-182), scale_c = f16(max_r |h[r,c]| / 8), codes
// packed COLUMN-major, i.e. nibble index c*rows + r (codec.py:232-233).
//
// Two kernels:
//   colstats<MAX>   -- (outlier.cu) one read of x (kept in L2 with evict_last),
//                      per-column abs-max as f16 bit patterns via per-CTA
//                      partials and a last-CTA-per-strip reduction;
//   channel_quant   -- re-reads x (L2-resident for activation-sized tensors),
//                      quantises a 64-column x 256-row block with 8 column
//                      scales held in registers, transposes row-major codes
//                      into column-major bytes with warp shuffles + a 2 KB
//                      shared-memory stage, writes 16-byte column runs.
//   channel_dequant -- the inverse transpose.
// Fast path needs cols % 8 == 0 and rows % 32 == 0; anything else goes to the
// generic kernels in group.cu.
#include "common.cuh"
#include "launch.h"

namespace adc {

constexpr int kTileCols = 64;     // 8 column units of 8
constexpr int kSubRows = 64;      // rows per sub-tile (32 row pairs)
constexpr int kBlockRows = 256;   // rows per block (4 sub-tiles)
constexpr int kWordStride = 9;    // padded smem stride (words) per column

// Byte `b` of word w.
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int b) { return (w >> (8 * b)) & 0xffu; }

// Raw input words of 8 elements, converted to f16 words on use.
template <int DT>
struct ChRaw {
  uint4 v;
  __device__ __forceinline__ void load(const void *x, int64_t i) {
    v = ld_stream16(static_cast<const char *>(x) + i * 2);
  }
  __device__ __forceinline__ void zero() { v = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ uint4 f16() const {
    if (DT == ADC_BF16) return make_uint4(bf2_to_h2(v.x), bf2_to_h2(v.y), bf2_to_h2(v.z), bf2_to_h2(v.w));
    return v;
  }
};
template <>
struct ChRaw<ADC_F32> {
  uint4 a, b;
  __device__ __forceinline__ void load(const void *x, int64_t i) {
    const char *p = static_cast<const char *>(x) + i * 4;
    a = ld_stream16(p);
    b = ld_stream16(p + 16);
  }
  __device__ __forceinline__ void zero() { a = b = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ uint4 f16() const {
    return make_uint4(f32x2_to_h2(__uint_as_float(a.x), __uint_as_float(a.y)),
                      f32x2_to_h2(__uint_as_float(a.z), __uint_as_float(a.w)),
                      f32x2_to_h2(__uint_as_float(b.x), __uint_as_float(b.y)),
                      f32x2_to_h2(__uint_as_float(b.z), __uint_as_float(b.w)));
  }
};

// Element pair (row r, row r+1) of column j of this thread's 8 columns as
// f32 for the packed quotient.  bf16 input goes straight to f32 (a shift or a
// mask): the f16 rounding the reference applies first cannot change a code
// once the column's scale is a normal f16 (every bf16 value at or above
// 2^-17 is exactly an f16; below it, the quotient stays under 1/2 either way),
// which the fast path requires anyway.
template <int DT>
__device__ __forceinline__ uint64_t col_pair(const ChRaw<DT> &ra, const ChRaw<DT> &rb, const uint4 &ha,
                                             const uint4 &hb, int j) {
  if constexpr (DT == ADC_BF16) {
    const uint32_t wa[4] = {ra.v.x, ra.v.y, ra.v.z, ra.v.w}, wb[4] = {rb.v.x, rb.v.y, rb.v.z, rb.v.w};
    const uint32_t a = (j & 1) ? (wa[j >> 1] & 0xffff0000u) : (wa[j >> 1] << 16);
    const uint32_t b = (j & 1) ? (wb[j >> 1] & 0xffff0000u) : (wb[j >> 1] << 16);
    return f2_pack(__uint_as_float(a), __uint_as_float(b));
  } else {
    const uint32_t wa[4] = {ha.x, ha.y, ha.z, ha.w}, wb[4] = {hb.x, hb.y, hb.z, hb.w};
    const uint32_t sh = (j & 1) * 16;
    return f2_pack(h2f((wa[j >> 1] >> sh) & 0xffffu), h2f((wb[j >> 1] >> sh) & 0xffffu));
  }
}

constexpr int kColBytes = 36;  // shared-memory bytes per tile column per sub-tile (32 row pairs + pad)

template <int DT>
__global__ void __launch_bounds__(kThreads)
    channel_quant(const void *__restrict__ x, int64_t rows, int64_t cols,
                  const uint32_t *__restrict__ colmax, uint8_t *__restrict__ codes,
                  uint16_t *__restrict__ scales) {
  // a programmatic dependent of the column abs-max pass (launch_k_dep): the
  // tile's rows are loaded before the wait (x is only read by that pass), the
  // column maxima after it
  // all four sub-tiles: their rows are loaded up front (8 x 16 B in flight per
  // thread, issued before the scales are derived), quantised, and their code
  // bytes written column-major into shared memory (one byte store per column
  // and row pair: the transpose), then stored as 16-byte column runs after one
  // barrier
  constexpr int kSubs = kBlockRows / kSubRows;
  __shared__ __align__(16) uint8_t stage[kSubs][kTileCols * kColBytes];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = lane & 7;         // column unit inside the tile
  const int tyl = lane >> 3;       // row pair inside the warp (0..3)
  const int rp = warp * 4 + tyl;   // row pair inside the sub-tile (0..31)
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kTileCols + tx * 8;
  const bool col_live = c0 < cols;
  const int64_t row_begin = static_cast<int64_t>(blockIdx.y) * kBlockRows;
  ChRaw<DT> ra[kSubs], rb[kSubs];
#pragma unroll
  for (int sub = 0; sub < kSubs; ++sub) {
    const int64_t r = row_begin + sub * kSubRows + 2 * rp;
    if (col_live && r < rows) {  // rows % 32 == 0 => r+1 < rows too
      ra[sub].load(x, r * cols + c0);
      rb[sub].load(x, (r + 1) * cols + c0);
    } else {
      ra[sub].zero();
      rb[sub].zero();
    }
  }
  pdl_wait();
  pdl_trigger();

  // Per-column quantisation constants for this thread's 8 columns.
  float qs[8], qi[8];
  bool fast = true;  // every column scale of this thread is a normal f16 (the packed path)
  {
    uint32_t sb[8];
    const uint4 m0 = col_live ? __ldg(reinterpret_cast<const uint4 *>(colmax + c0)) : make_uint4(0, 0, 0, 0);
    const uint4 m1 = col_live ? __ldg(reinterpret_cast<const uint4 *>(colmax + c0) + 1) : make_uint4(0, 0, 0, 0);
    const uint32_t top[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sb[j] = sym_scale_bits(top[j]);
      QParams q = make_qparams(static_cast<uint16_t>(sb[j]), 0);
      qs[j] = q.s;
      qi[j] = q.inv;
      fast &= (sb[j] & 0x7fffu) >= 0x0400u;
    }
    if (blockIdx.y == 0 && warp == 0 && tyl == 0 && col_live) {
      uint4 v = make_uint4(sb[0] | (sb[1] << 16), sb[2] | (sb[3] << 16), sb[4] | (sb[5] << 16),
                           sb[6] | (sb[7] << 16));
      *reinterpret_cast<uint4 *>(scales + c0) = v;
    }
  }

#pragma unroll
  for (int sub = 0; sub < kSubs; ++sub) {
    const uint4 ha = DT == ADC_BF16 ? make_uint4(0, 0, 0, 0) : ra[sub].f16();
    const uint4 hb = DT == ADC_BF16 ? make_uint4(0, 0, 0, 0) : rb[sub].f16();
    // byte j = code(row r, col j) | code(row r+1, col j) << 4
    uint32_t lo = 0, hi = 0;
    if (fast) {
      // rows r and r+1 of column j share its scale: one FMUL2 / two FFMA2
      // give both correctly rounded quotients, the magic add rounds them,
      // one saturating I2IP clips both and joins them into the byte, chained
      // four bytes per word (see pack8_tbits_sat)
      const uint64_t mg2 = f2_pack(kMagic8, kMagic8);
      uint32_t ta_[8], tb_[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint64_t h2 = col_pair<DT>(ra[sub], rb[sub], ha, hb, j);
        const uint64_t inv2 = f2_pack(qi[j], qi[j]), ns2 = f2_pack(-qs[j], -qs[j]);
        const uint64_t r0 = f2_mul(h2, inv2);
        const uint64_t r1 = f2_fma(f2_fma(r0, ns2, h2), inv2, r0);
        float ta, tb;
        f2_unpack(f2_add(r1, mg2), ta, tb);
        ta_[j] = __float_as_uint(ta) - 0x4B400008u;  // s32 codes
        tb_[j] = __float_as_uint(tb) - 0x4B400008u;
      }
      lo = pack4_pairs_sat(ta_, tb_);
      hi = pack4_pairs_sat(ta_ + 4, tb_ + 4);
    } else {
      const uint4 fa = ra[sub].f16(), fb = rb[sub].f16();  // the reference's f16 rounding
      uint32_t wa[4] = {fa.x, fa.y, fa.z, fa.w};
      uint32_t wb[4] = {fb.x, fb.y, fb.z, fb.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t sh = (j & 1) * 16;
        const float a = h2f((wa[j >> 1] >> sh) & 0xffffu);
        const float b = h2f((wb[j >> 1] >> sh) & 0xffffu);
        QParams q;
        q.s = qs[j];
        q.inv = qi[j];
        q.o = 0.f;
        const uint32_t byte = (static_cast<uint32_t>(sym_code(a, q)) & 0xfu) |
                              ((static_cast<uint32_t>(sym_code(b, q)) & 0xfu) << 4);
        if (j < 4)
          lo |= byte << (8 * j);
        else
          hi |= byte << (8 * (j - 4));
      }
    }
    // the transpose: byte j goes to column tx*8 + j, row pair rp
    uint8_t *sp = &stage[sub][(tx * 8) * kColBytes + rp];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sp[j * kColBytes] = static_cast<uint8_t>(lo >> (8 * j));
      sp[(j + 4) * kColBytes] = static_cast<uint8_t>(hi >> (8 * j));
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 2; ++q) {  // kSubs * kTileCols * 2 = 512 column runs of 16 B
    const int item = threadIdx.x + q * kThreads;
    const int sub = item / (kTileCols * 2), within = item % (kTileCols * 2);
    const int c = within >> 1, h = within & 1;
    const int64_t cg = static_cast<int64_t>(blockIdx.x) * kTileCols + c;
    const int64_t rs = row_begin + sub * kSubRows + 32 * h;
    if (cg < cols && rs < rows) {
      const uint32_t *sp = reinterpret_cast<const uint32_t *>(&stage[sub][c * kColBytes + 16 * h]);
      st_stream16(codes + (cg * rows + rs) / 2, make_uint4(sp[0], sp[1], sp[2], sp[3]));
    }
  }
}

template <int OT>
__global__ void __launch_bounds__(kThreads)
    channel_dequant(const uint8_t *__restrict__ codes, const uint16_t *__restrict__ scales,
                    int64_t rows, int64_t cols, void *__restrict__ y) {
  pdl_entry();
  // all four sub-tiles' column-major code runs are staged with one barrier
  // (2 x 16 B loads per thread in flight), then expanded without barriers
  constexpr int kSubs = kBlockRows / kSubRows;
  __shared__ uint32_t stage[kSubs][kTileCols * kWordStride];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = lane & 7, tyl = lane >> 3;
  const int rp = warp * 4 + tyl;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kTileCols + tx * 8;
  const bool col_live = c0 < cols;
  const int64_t row_begin = static_cast<int64_t>(blockIdx.y) * kBlockRows;
  {
    uint4 v[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int item = threadIdx.x + q * kThreads;  // kSubs * kTileCols * 2 = 512 items
      const int sub = item / (kTileCols * 2), within = item % (kTileCols * 2);
      const int c = within >> 1, h = within & 1;
      const int64_t cg = static_cast<int64_t>(blockIdx.x) * kTileCols + c;
      const int64_t rs = row_begin + sub * kSubRows + 32 * h;
      v[q] = (cg < cols && rs < rows) ? ld_stream16(codes + (cg * rows + rs) / 2) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int item = threadIdx.x + q * kThreads;
      const int sub = item / (kTileCols * 2), within = item % (kTileCols * 2);
      uint32_t *s = &stage[sub][(within >> 1) * kWordStride + 4 * (within & 1)];
      s[0] = v[q].x;
      s[1] = v[q].y;
      s[2] = v[q].z;
      s[3] = v[q].w;
    }
  }
  float sc[8];
  {
    uint4 v = col_live ? __ldg(reinterpret_cast<const uint4 *>(scales + c0)) : make_uint4(0, 0, 0, 0);
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) sc[j] = h2f((w[j >> 1] >> ((j & 1) * 16)) & 0xffffu);
  }
  __syncthreads();
#pragma unroll
  for (int sub = 0; sub < kSubs; ++sub) {
    const int64_t r = row_begin + sub * kSubRows + 2 * rp;
    if (!col_live || r >= rows) continue;
    float va[8], vb[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t word = stage[sub][(tx * 8 + j) * kWordStride + warp];
      const uint32_t byte = byte_of(word, tyl);
      va[j] = nib_code(byte, 0) * sc[j];
      vb[j] = nib_code(byte, 1) * sc[j];
    }
    Storer<OT>::store8(y, r * cols + c0, va);
    Storer<OT>::store8(y, (r + 1) * cols + c0, vb);
  }
}

#define ADC_DT_SWITCH(dt, DT, ...)                                   \
  switch (dt) {                                                      \
    case ADC_F32: { constexpr int DT = ADC_F32; __VA_ARGS__; break; }  \
    case ADC_BF16: { constexpr int DT = ADC_BF16; __VA_ARGS__; break; } \
    case ADC_F16: { constexpr int DT = ADC_F16; __VA_ARGS__; break; }  \
    default: return -1;                                              \
  }

static inline bool al(const void *p, size_t a) { return reinterpret_cast<uintptr_t>(p) % a == 0; }

bool channel_fast_ok(const void *x, int64_t rows, int64_t cols, const void *codes,
                     const void *scales) {
  return cols % 8 == 0 && rows % 32 == 0 && al(x, 16) && al(codes, 16) && al(scales, 16);
}

int launch_channel_compress(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                            const Workspace &ws, uint8_t *codes, uint16_t *scales,
                            uint32_t *err) {
  if (launch_colstats_max(c, x, dt, rows, cols, ws, err)) return -1;
  dim3 gq(static_cast<unsigned>((cols + kTileCols - 1) / kTileCols),
          static_cast<unsigned>((rows + kBlockRows - 1) / kBlockRows));
  ADC_DT_SWITCH(dt, DT, {
    launch_k_dep(channel_quant<DT>, gq, kThreads, 0, c.stream, x, rows, cols, ws.colmax, codes, scales), note_launches(1);
  });
  return 0;
}

int launch_channel_decompress(const Ctx &c, const uint8_t *codes, const uint16_t *scales,
                              int64_t rows, int64_t cols, void *y, int ot) {
  dim3 g(static_cast<unsigned>((cols + kTileCols - 1) / kTileCols),
         static_cast<unsigned>((rows + kBlockRows - 1) / kBlockRows));
  switch (ot) {
    case ADC_F32: launch_k(channel_dequant<ADC_F32>, g, kThreads, 0, c.stream, codes, scales, rows, cols, y), note_launches(1); break;
    case ADC_BF16: launch_k(channel_dequant<ADC_BF16>, g, kThreads, 0, c.stream, codes, scales, rows, cols, y), note_launches(1); break;
    case ADC_F16: launch_k(channel_dequant<ADC_F16>, g, kThreads, 0, c.stream, codes, scales, rows, cols, y), note_launches(1); break;
    default: return -1;
  }
  return 0;
}

}  // namespace adc
