// Host-side launchers shared between the kernel translation units and the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace adc {

// 32-bit division by a runtime constant: q = (n * m) >> p, exact for n < 2^31.
struct FastDiv {
  uint64_t m;
  uint32_t p;
  uint32_t d;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.p = 31 + l;
  f.m = ((1ull << f.p) + d - 1) / d;  // ceil(2^p / d)
  return f;
}

// Count of kernels this library has launched (adc_kernel_launches()).
void note_launches(int n);

// Kernel launches go through launch_k: cudaLaunchKernelEx with programmatic
// stream serialisation (PDL, see pdl_entry() in common.cuh) when enabled by
// ADC_PDL=1 / adc_set_option("pdl", 1).
bool pdl_enabled();
void set_pdl(int v);
void set_cr_rows8(int v);
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// The zeroing quantiser of the outlier-separated path is launched as a
// programmatic dependent of the column statistics (always, unless
// adc_set_option("outlier_pdl", 0)): the statistics kernel triggers its
// dependents once every CTA has added its column partials, so the
// quantiser's CTAs start, and issue their first x loads (x is not written by
// the statistics kernel), while the last statistics CTA computes mean / std /
// flags; griddepcontrol.wait then orders every read of the flags.  The
// per-channel quantiser follows the column abs-max pass the same way.
bool outlier_pdl_enabled();
void set_outlier_pdl(int v);
template <typename... KArgs, typename... Args>
inline void launch_k_dep(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                         Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_enabled() || outlier_pdl_enabled()) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

struct Ctx {
  cudaStream_t stream;
  int num_sms;
};

// Workspace carving (offsets in bytes, 256-aligned).  Must be zero-filled
// once by the caller; the kernels leave every counter at zero on exit.
struct Workspace {
  double *colsum;        // cols       column |x| sums (outlier)
  uint32_t *colmax;      // cols       column abs-max f16 bits (per-channel)
  uint8_t *flag;         // cols + 8   outlier flags
  double *acc;           // cols       f64 atomic column-sum accumulators (zero at rest)
  double *k4acc;         // 2 x cols   single-pass kernel's bulk-reduction targets (double-buffered)
  uint32_t *macc;        // cols       u32 atomic column-max accumulators (zero at rest)
  uint32_t *counters;    // 8          arrival counters ([0..3] colreduce, [4..7] k4: barrier count / base / epoch / layout)
  uint8_t *pflag;        // cols + 8   previous outlier flags (the single pass's prediction; any
                         //            content is valid, zero-fill = "no outliers")
  int32_t *node_lo;      // pairwise-tree nodes (used when cols > 16384)
  int32_t *node_n;
  int32_t *node_left;
  double *node_val;
  size_t bytes;
};

size_t workspace_layout(int64_t cols, Workspace *ws, void *base);

// group kernels (group.cu)
int launch_group_compress(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                          int64_t g, bool asym, const uint8_t *zero_flag, const uint32_t *idx, const int32_t *k_dev, uint16_t *outl_val,
                          int64_t k_cap, uint8_t *codes, uint16_t *scales, uint16_t *offsets,
                          uint32_t *err, const uint32_t *requant = nullptr);
int launch_group_decompress(const Ctx &c, const uint8_t *codes, const uint16_t *scales,
                            const uint16_t *offsets, int64_t rows, int64_t cols, int64_t g,
                            bool asym, void *y, int ot);
// one-launch outlier decompress (shared-memory tiles); returns 1 when not eligible
int launch_outlier_decompress_tiles(const Ctx &c, const uint8_t *codes, const uint16_t *scales,
                                   const uint32_t *idx, const uint16_t *val, const int32_t *k_dev,
                                   int64_t k_cap, int64_t rows, int64_t cols, int64_t g, void *y,
                                   int ot);
void set_outlier_decompress_mode(int m);
void set_outlier_tile(int t);
void set_cr_trace(int v);
void set_sum_smem_cols(int v);
int read_cr_trace(unsigned long long *host, int n);
int launch_outlier_scatter(const Ctx &c, const uint32_t *idx, const uint16_t *val,
                           const int32_t *k_dev, int64_t k_cap, int64_t rows, int64_t cols,
                           void *y, int ot, const uint8_t *codes = nullptr,
                           const uint16_t *scales = nullptr, int64_t g = 0);

bool use_epl32();
void set_epl(int v);

int launch_outlier_gather(const Ctx &c, const void *x, int dt, const uint32_t *idx,
                          const int32_t *k_dev, int64_t k_cap, int64_t rows, int64_t cols,
                          uint16_t *outl_val);

// single-pass outlier-separated compress (k4.cu): returns 1 if it ran, 0 if
// the shape is not eligible or not selected (ADC_OUTLIER_PATH /
// adc_set_option("outlier_path", 0 two launches | 1 single pass | 2 auto)); the
// caller then uses the colreduce + group_quant_fast pair (identical bytes).
int launch_outlier_k4(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols, int64_t g,
                      double thr, int64_t k_cap, const Workspace &ws, uint8_t *codes,
                      uint16_t *scales, uint32_t *idx, uint16_t *val, int32_t *k_out,
                      uint32_t *err);
int k4_mode();
void set_k4_mode(int v);
void set_k4_trace(int v);
void set_k4_dbg(int v);
int read_k4_trace(unsigned long long *host, int n);
// int8 extension (int8.cu; parity unpinned, oracle/int8_oracle.py)
int launch_int8_compress(const Ctx &c, const void *x, int dt, int64_t n, int64_t g, int8_t *codes,
                         float *scales, uint32_t *err);
int launch_int8_decompress(const Ctx &c, const int8_t *codes, const float *scales, int64_t n, int64_t g,
                           void *y, int ot);
int launch_int4f32_compress(const Ctx &c, const void *x, int dt, int64_t n, int64_t g, uint8_t *codes,
                            float *scales, uint32_t *err);
int launch_int4f32_decompress(const Ctx &c, const uint8_t *codes, const float *scales, int64_t n, int64_t g,
                              void *y, int ot);

// device-side ADC1 serialisation (wire.cu)
int launch_wire_serialize(const Ctx &c, int scheme, int64_t rows, int64_t cols, int64_t group,
                          int64_t n_groups, const uint16_t *scales, const uint16_t *offsets,
                          const uint8_t *codes, int64_t code_bytes, const uint32_t *idx,
                          const uint16_t *val, const int32_t *k_dev, int64_t k_cap, uint8_t *out,
                          int64_t out_cap, uint64_t *out_len, uint32_t *err);
int launch_wire_deserialize(const Ctx &c, const uint8_t *in, int scheme, int64_t rows, int64_t cols,
                            int64_t n_groups, int64_t code_bytes, int64_t k, uint16_t *scales,
                            uint16_t *offsets, uint8_t *codes, uint32_t *idx, uint16_t *val, uint32_t *err);

// per-channel kernels (channel.cu)
bool channel_fast_ok(const void *x, int64_t rows, int64_t cols, const void *codes,
                     const void *scales);
int launch_channel_compress(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                            const Workspace &ws, uint8_t *codes, uint16_t *scales,
                            uint32_t *err);
int launch_channel_decompress(const Ctx &c, const uint8_t *codes, const uint16_t *scales,
                              int64_t rows, int64_t cols, void *y, int ot);

// column statistics (outlier.cu): one launch each
int launch_colstats_sum(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                        const Workspace &ws, bool do_stats, double thr, int64_t k_cap,
                        uint32_t *idx, int32_t *k_out, uint32_t *err, bool too_many_check);
int launch_colstats_max(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                        const Workspace &ws, uint32_t *err);

// masks (mask.cu)
int launch_mask_pack(const Ctx &c, const void *m, int dt, int64_t n, uint8_t *bits,
                     uint32_t *err);
int launch_mask_unpack(const Ctx &c, const uint8_t *bits, int64_t n, uint8_t *out);

}  // namespace adc
