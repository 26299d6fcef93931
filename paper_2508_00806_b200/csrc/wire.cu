// Device-side ADC1 serialisation: the reference's wire
// format (serialize, codec.py:432-459) assembled straight from the device
// payload, without a round trip through host memory:
//   25-byte header <4sBIIIII: "ADC1", scheme, rows, cols, group_size,
//   group_count, k>; per-group float16 scales (asymmetric: interleaved
//   [scale, offset] pairs); packed codes (mask bits for BIT_MASK); k u32
//   indices; k x rows float16 outlier values.
// k comes from the device (written by adc_compress), so the segment offsets
// are computed on the device too; the total length is written to *out_len.
// Each thread assembles 16 output bytes (one aligned 128-bit store) from the
// segments by byte gathers -- the header makes every later segment unaligned.
#include "common.cuh"
#include "launch.h"

namespace adc {

struct WireArgs {
  int scheme;
  uint32_t rows, cols, group, n_groups;
  const uint16_t *scales, *offsets;
  const uint8_t *codes;
  uint64_t code_bytes;
  const uint32_t *idx;
  const uint16_t *val;
  const int32_t *k_dev;
  int64_t k_cap;
  uint8_t *out;
  uint64_t out_cap;
  uint64_t *out_len;
  uint32_t *err;
};

__device__ __forceinline__ uint8_t wire_byte(const WireArgs &a, uint64_t p, uint64_t k, uint64_t m0,
                                             uint64_t c0, uint64_t i0, uint64_t v0, uint64_t end) {
  if (p < 25) {
    if (p < 4) return static_cast<uint8_t>("ADC1"[p]);
    if (p == 4) return static_cast<uint8_t>(a.scheme);
    const uint32_t f = static_cast<uint32_t>((p - 5) / 4), sh = 8 * static_cast<uint32_t>((p - 5) % 4);
    const uint32_t v = f == 0 ? a.rows : f == 1 ? a.cols : f == 2 ? a.group : f == 3 ? a.n_groups
                                                                                     : static_cast<uint32_t>(k);
    return static_cast<uint8_t>(v >> sh);
  }
  if (p < c0) {  // group metadata
    const uint64_t q = p - m0;
    if (a.offsets) {  // [scale, offset] pairs
      const uint64_t gidx = q / 4, r = q % 4;
      const uint16_t h = r < 2 ? a.scales[gidx] : a.offsets[gidx];
      return static_cast<uint8_t>(h >> (8 * (r & 1)));
    }
    return static_cast<uint8_t>(a.scales[q / 2] >> (8 * (q & 1)));
  }
  if (p < i0) return a.codes[p - c0];
  if (p < v0) {
    const uint64_t q = p - i0;
    return static_cast<uint8_t>(a.idx[q / 4] >> (8 * (q % 4)));
  }
  if (p < end) {
    const uint64_t q = p - v0;
    return static_cast<uint8_t>(a.val[q / 2] >> (8 * (q & 1)));
  }
  return 0;
}

__global__ void __launch_bounds__(kThreads) wire_serialize(WireArgs a) {
  pdl_entry();
  const uint64_t k = a.k_dev ? static_cast<uint64_t>(min(static_cast<int64_t>(*a.k_dev), a.k_cap)) : 0;
  const uint64_t meta = a.scheme == ADC_BIT_MASK ? 0 : static_cast<uint64_t>(a.n_groups) * (a.offsets ? 4 : 2);
  const uint64_t m0 = 25, c0 = m0 + meta, i0 = c0 + a.code_bytes, v0 = i0 + 4 * k,
                 end = v0 + 2 * k * a.rows;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.out_len = end;
    if (end > a.out_cap && a.err) atomicOr(a.err, ADC_ERR_K_CAP);
  }
  const uint64_t lim = min(end, a.out_cap);
  const uint64_t chunks = (lim + 15) / 16;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; t < chunks;
       t += static_cast<uint64_t>(gridDim.x) * kThreads) {
    const uint64_t p0 = 16 * t;
    uint32_t w[4] = {0, 0, 0, 0};
    if (p0 >= c0 && p0 + 16 <= i0) {
      // inside the code segment: byte loads from a contiguous source
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j >> 2] |= static_cast<uint32_t>(a.codes[p0 + j - c0]) << (8 * (j & 3));
    } else {
#pragma unroll 4
      for (int j = 0; j < 16; ++j)
        if (p0 + j < lim) w[j >> 2] |= static_cast<uint32_t>(wire_byte(a, p0 + j, k, m0, c0, i0, v0, end)) << (8 * (j & 3));
    }
    if (p0 + 16 <= lim) {
      *reinterpret_cast<uint4 *>(a.out + p0) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (int j = 0; p0 + j < lim; ++j) a.out[p0 + j] = static_cast<uint8_t>(w[j >> 2] >> (8 * (j & 3)));
    }
  }
}

int launch_wire_serialize(const Ctx &c, int scheme, int64_t rows, int64_t cols, int64_t group,
                          int64_t n_groups, const uint16_t *scales, const uint16_t *offsets,
                          const uint8_t *codes, int64_t code_bytes, const uint32_t *idx,
                          const uint16_t *val, const int32_t *k_dev, int64_t k_cap, uint8_t *out,
                          int64_t out_cap, uint64_t *out_len, uint32_t *err) {
  WireArgs a{scheme, static_cast<uint32_t>(rows), static_cast<uint32_t>(cols), static_cast<uint32_t>(group),
             static_cast<uint32_t>(n_groups), scales, offsets, codes, static_cast<uint64_t>(code_bytes),
             idx, val, k_dev, k_cap, out, static_cast<uint64_t>(out_cap), out_len, err};
  const int64_t chunks = (out_cap + 15) / 16;
  int64_t grid = (chunks + kThreads - 1) / kThreads;
  const int64_t cap = static_cast<int64_t>(c.num_sms) * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  launch_k(wire_serialize, dim3(static_cast<unsigned>(grid)), dim3(kThreads), 0, c.stream, a);
  note_launches(1);
  return 0;
}

// ---------------------------------------------------------------------------
// Device-side ADC1 deserialisation: the content half of the reference's
// validator (deserialize, codec.py:506-546) plus the split of the payload
// into the record's device arrays.  The header half (magic, scheme, shape,
// counts, total length; codec.py:464-493) is adc_parse_header on the host --
// it decides the output sizes.  One thread per output unit:
//   group g          -> scale (and offset) bytes, checked finite / >= 0
//   16 code bytes    -> one aligned 128-bit store (unaligned byte gathers)
//   outlier rank j   -> index, checked < cols and > index j-1
//   8 value halves   -> 16-byte store
// Violations OR ADC_ERR_BAD_* bits into err (the host raises them in the
// reference's order: scales, offsets, index range, index order).
struct UnwireArgs {
  const uint8_t *in;
  uint64_t n_groups, code_bytes, k, n_vals;
  uint64_t m0, c0, i0, v0;  // segment offsets in the payload
  uint32_t cols;
  int asym;
  uint16_t *scales, *offsets;
  uint8_t *codes;
  uint32_t *idx;
  uint16_t *val;
  uint32_t *err;
};

__device__ __forceinline__ uint16_t ld_u16(const uint8_t *p) {
  return static_cast<uint16_t>(p[0] | (static_cast<uint32_t>(p[1]) << 8));
}

__device__ __forceinline__ uint32_t ld_u32(const uint8_t *p) {
  return p[0] | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}

__global__ void __launch_bounds__(kThreads) wire_deserialize(UnwireArgs a) {
  pdl_entry();
  const uint64_t code_units = (a.code_bytes + 15) / 16, val_units = (a.n_vals + 7) / 8;
  const uint64_t e0 = a.n_groups, e1 = e0 + code_units, e2 = e1 + a.k, e3 = e2 + val_units;
  uint32_t bad = 0;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; t < e3;
       t += static_cast<uint64_t>(gridDim.x) * kThreads) {
    if (t < e0) {
      const uint8_t *p = a.in + a.m0 + t * (a.asym ? 4 : 2);
      const uint16_t s = ld_u16(p);
      // not finite: exponent all ones; negative: sign set on a non-zero value
      if ((s & 0x7c00u) == 0x7c00u || ((s & 0x8000u) && (s & 0x7fffu))) bad |= ADC_ERR_BAD_SCALE;
      a.scales[t] = s;
      if (a.asym) {
        const uint16_t o = ld_u16(p + 2);
        if ((o & 0x7c00u) == 0x7c00u) bad |= ADC_ERR_BAD_OFFSET;
        a.offsets[t] = o;
      }
    } else if (t < e1) {
      const uint64_t q = 16 * (t - e0);
      const uint8_t *p = a.in + a.c0 + q;
      if (q + 16 <= a.code_bytes) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = ld_u32(p + 4 * j);
        *reinterpret_cast<uint4 *>(a.codes + q) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
        for (uint64_t j = 0; q + j < a.code_bytes; ++j) a.codes[q + j] = p[j];
      }
    } else if (t < e2) {
      const uint64_t j = t - e1;
      const uint32_t v = ld_u32(a.in + a.i0 + 4 * j);
      if (v >= a.cols) bad |= ADC_ERR_BAD_INDEX_RANGE;
      if (j > 0 && v <= ld_u32(a.in + a.i0 + 4 * (j - 1))) bad |= ADC_ERR_BAD_INDEX_ORDER;
      a.idx[j] = v;
    } else {
      const uint64_t q = 8 * (t - e2);
      const uint8_t *p = a.in + a.v0 + 2 * q;
      for (uint64_t j = 0; j < 8 && q + j < a.n_vals; ++j) a.val[q + j] = ld_u16(p + 2 * j);
    }
  }
  if (bad) atomicOr(a.err, bad);
}

int launch_wire_deserialize(const Ctx &c, const uint8_t *in, int scheme, int64_t rows, int64_t cols,
                            int64_t n_groups, int64_t code_bytes, int64_t k, uint16_t *scales,
                            uint16_t *offsets, uint8_t *codes, uint32_t *idx, uint16_t *val, uint32_t *err) {
  const bool asym = scheme == ADC_ASYMMETRIC_GROUP;
  const uint64_t m0 = 25, c0 = m0 + static_cast<uint64_t>(n_groups) * (asym ? 4 : 2);
  const uint64_t i0 = c0 + static_cast<uint64_t>(code_bytes), v0 = i0 + 4 * static_cast<uint64_t>(k);
  UnwireArgs a{in, static_cast<uint64_t>(n_groups), static_cast<uint64_t>(code_bytes), static_cast<uint64_t>(k),
               static_cast<uint64_t>(k) * static_cast<uint64_t>(rows), m0, c0, i0, v0,
               static_cast<uint32_t>(cols), asym ? 1 : 0, scales, offsets, codes, idx, val, err};
  const uint64_t units = a.n_groups + (a.code_bytes + 15) / 16 + a.k + (a.n_vals + 7) / 8;
  int64_t grid = static_cast<int64_t>((units + kThreads - 1) / kThreads);
  const int64_t cap = static_cast<int64_t>(c.num_sms) * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  launch_k(wire_deserialize, dim3(static_cast<unsigned>(grid)), dim3(kThreads), 0, c.stream, a);
  note_launches(1);
  return 0;
}

}  // namespace adc
