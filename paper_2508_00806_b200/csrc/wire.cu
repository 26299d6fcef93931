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

}  // namespace adc
