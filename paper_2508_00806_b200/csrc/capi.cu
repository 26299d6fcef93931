// C-ABI entry points (include/adacc.h): argument validation, workspace
// carving and kernel dispatch.  No allocation, no synchronisation.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "launch.h"

namespace adc {

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};

static std::atomic<int> g_pdl{-1};
bool pdl_enabled() {
  int v = g_pdl.load(std::memory_order_relaxed);
  if (v < 0) {
    // measured on the bench step (CUDA graph of 18 codec calls): 3538 GB/s
    // with PDL vs 3561 without, so it is off unless ADC_PDL=1
    const char *e = getenv("ADC_PDL");
    v = (e && e[0] == '1') ? 1 : 0;
    g_pdl.store(v, std::memory_order_relaxed);
  }
  return v == 1;
}
void set_pdl(int v) { g_pdl.store(v ? 1 : 0, std::memory_order_relaxed); }
static std::atomic<int> g_outlier_pdl{1};
bool outlier_pdl_enabled() { return g_outlier_pdl.load(std::memory_order_relaxed) != 0; }
void set_outlier_pdl(int v) { g_outlier_pdl.store(v ? 1 : 0, std::memory_order_relaxed); }

void note_launches(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n), std::memory_order_relaxed); }

static int fail(int code, const char *msg) {
  g_last_error = msg;
  return code;
}

static int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return ADC_ECUDA;
  }
  g_last_error.clear();
  return ADC_OK;
}

static int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

static inline size_t up256(size_t v) { return (v + 255) & ~size_t(255); }

static int64_t node_capacity(int64_t cols) { return cols / 16 + 64; }

size_t workspace_layout(int64_t cols, Workspace *ws, void *base) {
  char *p = static_cast<char *>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *r = p ? p + off : nullptr;
    off += up256(bytes);
    return r;
  };
  Workspace w;
  const int64_t nodes = node_capacity(cols);
  w.counters = reinterpret_cast<uint32_t *>(take(sizeof(uint32_t) * 8));
  w.colsum = reinterpret_cast<double *>(take(sizeof(double) * cols));
  w.colmax = reinterpret_cast<uint32_t *>(take(sizeof(uint32_t) * cols));
  w.flag = reinterpret_cast<uint8_t *>(take(static_cast<size_t>(cols) + 8));
  w.node_lo = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * nodes));
  w.node_n = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * nodes));
  w.node_left = reinterpret_cast<int32_t *>(take(sizeof(int32_t) * nodes));
  w.node_val = reinterpret_cast<double *>(take(sizeof(double) * nodes));
  w.acc = reinterpret_cast<double *>(take(sizeof(double) * cols));
  w.k4acc = reinterpret_cast<double *>(take(sizeof(double) * 2 * cols));
  w.macc = reinterpret_cast<uint32_t *>(take(sizeof(uint32_t) * cols));
  w.pflag = reinterpret_cast<uint8_t *>(take(static_cast<size_t>(cols) + 8));
  w.bytes = off;
  if (ws) *ws = w;
  return off;
}

static bool valid_float_dtype(int dt) { return dt == ADC_F32 || dt == ADC_BF16 || dt == ADC_F16; }

}  // namespace adc

using namespace adc;

extern "C" {

const char *adc_version(void) { return "adacc-b200 0.1.0 (sm_100a)"; }

int adc_abi_version(void) { return ADC_ABI_VERSION; }

const char *adc_last_error(void) { return g_last_error.c_str(); }

unsigned long long adc_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

static int g_trace_src = 0;  // adc_debug_trace_k4 source: 0 single pass, 1 column statistics

int adc_set_option(const char *key, int value) {
  if (!key) return fail(ADC_EINVAL, "null option key");
  const std::string k(key);
  if (k == "pdl") {  // programmatic dependent launch on (1) / off (0, default)
    set_pdl(value);
    return ADC_OK;
  }
  if (k == "outlier_pdl") {  // zeroing quantiser as a programmatic dependent of the statistics (1, default)
    set_outlier_pdl(value);
    return ADC_OK;
  }
  if (k == "cr_rows8") {  // column pass grid: 0 one full wave, 1 >= 8 rows per row lane, 2 (default) + whole batches
    set_cr_rows8(value);
    return ADC_OK;
  }
  if (k == "epl") {  // elements per lane of the group quantiser: 32 (default) or 16
    set_epl(value);
    return ADC_OK;
  }
  if (k == "outlier_path") {  // 0: colreduce + quantiser, 1: single pass where eligible, 2: automatic (default)
    set_k4_mode(value);
    return ADC_OK;
  }
  if (k == "outlier_decompress") {  // 0: dequantise + overwrite launches, 2: one launch where eligible (default)
    set_outlier_decompress_mode(value);
    return ADC_OK;
  }
  if (k == "outlier_tile") {  // elements per tile of the one-launch outlier decompress: 4096, 8192 (default), 16384
    set_outlier_tile(value);
    return ADC_OK;
  }
  if (k == "k4_dbg") {  // timing experiments on the single-pass kernel (results invalid when != 0)
    set_k4_dbg(value);
    return ADC_OK;
  }
  if (k == "sum_smem_cols") {  // column statistics keep the sums in shared memory up to this many columns (8192)
    set_sum_smem_cols(value);
    return ADC_OK;
  }
  if (k == "cr_trace") {  // record phase timestamps of the column-statistics kernel (adc_debug_trace_k4 reads them)
    set_cr_trace(value);
    g_trace_src = value ? 1 : 0;
    return ADC_OK;
  }
  if (k == "k4_trace") {  // record phase timestamps of the single-pass kernel (adc_debug_trace_k4)
    set_k4_trace(value);
    return ADC_OK;
  }
  return fail(ADC_EINVAL, "unknown option");
}


int adc_debug_trace_k4(unsigned long long *out, int n) {
  if (!out || n < 0) return fail(ADC_EINVAL, "bad trace buffer");
  const int r = g_trace_src == 1 ? read_cr_trace(out, n) : read_k4_trace(out, n);
  return r < 0 ? fail(ADC_ECUDA, "trace copy failed") : r;
}

int adc_payload_bytes(int scheme, int64_t rows, int64_t cols, int64_t group_size,
                      int64_t outlier_count, int64_t *n_groups, int64_t *code_bytes,
                      int64_t *payload_bytes) {
  if (scheme < 0 || scheme > 3) return fail(ADC_EINVAL, "unknown scheme");
  if (rows < 1 || cols < 1) return fail(ADC_EINVAL, "shape must be at least 1x1");
  const int64_t n = rows * cols;
  int64_t groups = 0, codes = 0, total = 0;
  if (scheme == ADC_BIT_MASK) {
    codes = (n + 7) / 8;
    total = codes;
  } else {
    if (group_size < 0) return fail(ADC_EINVAL, "group_size must be positive or PER_CHANNEL");
    groups = group_size == ADC_PER_CHANNEL ? cols : (n + group_size - 1) / group_size;
    codes = (n + 1) / 2;
    total = (scheme == ADC_ASYMMETRIC_GROUP ? 4 : 2) * groups + codes;
    if (scheme == ADC_OUTLIER_SEPARATED) total += outlier_count * (4 + 2 * rows);
  }
  if (n_groups) *n_groups = groups;
  if (code_bytes) *code_bytes = codes;
  if (payload_bytes) *payload_bytes = total;
  return ADC_OK;
}

size_t adc_workspace_bytes(int scheme, int64_t rows, int64_t cols, int64_t group_size) {
  (void)scheme;
  (void)rows;
  (void)group_size;
  if (cols < 1) cols = 1;
  return workspace_layout(cols, nullptr, nullptr);
}

int adc_compress(int scheme, const void *x, int in_dtype, int64_t rows, int64_t cols,
                 int64_t group_size, double z_threshold, int64_t k_cap, uint8_t *codes,
                 uint16_t *scales, uint16_t *offsets, uint32_t *outlier_idx, uint16_t *outlier_val,
                 int32_t *k_out, uint32_t *err_word, void *workspace, size_t workspace_bytes,
                 void *stream) {
  if (scheme < 0 || scheme > 3) return fail(ADC_EINVAL, "unknown scheme");
  if (rows < 1 || cols < 1) return fail(ADC_EINVAL, "activation matrix must have at least one element");
  if (!x || !codes) return fail(ADC_EINVAL, "null input or code buffer");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  const int64_t n = rows * cols;
  if (scheme == ADC_BIT_MASK) {
    if (!(valid_float_dtype(in_dtype) || in_dtype == ADC_U8)) return fail(ADC_EINVAL, "bad mask dtype");
    if (launch_mask_pack(c, x, in_dtype, n, codes, err_word)) return fail(ADC_EINVAL, "mask dispatch");
    return check_launch("mask_pack");
  }
  if (!valid_float_dtype(in_dtype)) return fail(ADC_EINVAL, "activation dtype must be f32, bf16 or f16");
  if (group_size != ADC_PER_CHANNEL && group_size < 1)
    return fail(ADC_EINVAL, "group_size must be positive or PER_CHANNEL");
  if (!scales) return fail(ADC_EINVAL, "null scale buffer");
  if (scheme == ADC_ASYMMETRIC_GROUP && !offsets) return fail(ADC_EINVAL, "null offset buffer");
  const bool asym = scheme == ADC_ASYMMETRIC_GROUP;
  const bool pc = group_size == ADC_PER_CHANNEL;
  int rc = 0;
  if (scheme == ADC_OUTLIER_SEPARATED) {
    if (!k_out || (k_cap > 0 && (!outlier_idx || !outlier_val)))
      return fail(ADC_EINVAL, "outlier buffers required");
    if (!workspace || workspace_bytes < workspace_layout(cols, nullptr, nullptr))
      return fail(ADC_EWORKSPACE, "workspace too small");
    Workspace ws;
    workspace_layout(cols, &ws, workspace);
    if (launch_outlier_k4(c, x, in_dtype, rows, cols, group_size, z_threshold, k_cap, ws, codes, scales,
                          outlier_idx, outlier_val, k_out, err_word))
      return check_launch("outlier_single_pass");
    rc |= launch_colstats_sum(c, x, in_dtype, rows, cols, ws, true, z_threshold, k_cap,
                              outlier_idx, k_out, err_word, true);
    rc |= launch_group_compress(c, x, in_dtype, rows, cols, group_size, false, ws.flag,
                                outlier_idx, k_out, outlier_val, k_cap, codes, scales, nullptr,
                                err_word);
    if (rc) return fail(ADC_EINVAL, "outlier dispatch");
    return check_launch("outlier_separated");
  }
  if (pc && !asym && channel_fast_ok(x, rows, cols, codes, scales)) {
    if (!workspace || workspace_bytes < workspace_layout(cols, nullptr, nullptr))
      return fail(ADC_EWORKSPACE, "workspace too small");
    Workspace ws;
    workspace_layout(cols, &ws, workspace);
    if (launch_channel_compress(c, x, in_dtype, rows, cols, ws, codes, scales, err_word))
      return fail(ADC_EINVAL, "channel dispatch");
    return check_launch("per_channel");
  }
  rc = launch_group_compress(c, x, in_dtype, rows, cols, group_size, asym, nullptr, nullptr,
                             nullptr, nullptr, 0, codes, scales, offsets, err_word);
  if (rc) return fail(ADC_EINVAL, "group dispatch");
  return check_launch("group_quant");
}

int adc_decompress(int scheme, const uint8_t *codes, const uint16_t *scales,
                   const uint16_t *offsets, const uint32_t *outlier_idx,
                   const uint16_t *outlier_val, const int32_t *k_dev, int64_t k_cap, int64_t rows,
                   int64_t cols, int64_t group_size, void *y, int out_dtype, void *stream) {
  if (scheme < 0 || scheme > 3) return fail(ADC_EINVAL, "unknown scheme");
  if (rows < 1 || cols < 1) return fail(ADC_EINVAL, "bad shape");
  if (!codes || !y) return fail(ADC_EINVAL, "null buffer");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  const int64_t n = rows * cols;
  if (scheme == ADC_BIT_MASK) {
    if (out_dtype != ADC_U8) return fail(ADC_EINVAL, "masks decompress to u8");
    launch_mask_unpack(c, codes, n, static_cast<uint8_t *>(y));
    return check_launch("mask_unpack");
  }
  if (!valid_float_dtype(out_dtype)) return fail(ADC_EINVAL, "output dtype must be f32, bf16 or f16");
  if (group_size != ADC_PER_CHANNEL && group_size < 1) return fail(ADC_EINVAL, "bad group_size");
  if (!scales) return fail(ADC_EINVAL, "null scales");
  const bool asym = scheme == ADC_ASYMMETRIC_GROUP;
  if (asym && !offsets) return fail(ADC_EINVAL, "null offsets");
  const bool pc = group_size == ADC_PER_CHANNEL;
  int rc = 0;
  if (scheme == ADC_OUTLIER_SEPARATED && k_cap > 0 && !pc && outlier_idx && outlier_val && k_dev &&
      launch_outlier_decompress_tiles(c, codes, scales, outlier_idx, outlier_val, k_dev, k_cap, rows, cols,
                                     group_size, y, out_dtype) == 0)
    return check_launch("decompress");
  if (pc && !asym && channel_fast_ok(y, rows, cols, codes, scales) &&
      reinterpret_cast<uintptr_t>(y) % 16 == 0) {
    rc = launch_channel_decompress(c, codes, scales, rows, cols, y, out_dtype);
  } else {
    rc = launch_group_decompress(c, codes, scales, asym ? offsets : nullptr, rows, cols, group_size,
                                 asym, y, out_dtype);
  }
  if (rc) return fail(ADC_EINVAL, "decompress dispatch");
  if (scheme == ADC_OUTLIER_SEPARATED && k_cap > 0) {
    if (!outlier_idx || !outlier_val || !k_dev) return fail(ADC_EINVAL, "outlier buffers required");
    launch_outlier_scatter(c, outlier_idx, outlier_val, k_dev, k_cap, rows, cols, y, out_dtype,
                           pc ? nullptr : codes, scales, group_size);
  }
  return check_launch("decompress");
}

int adc_compress_int8(const void *x, int in_dtype, int64_t rows, int64_t cols, int64_t group_size,
                      int8_t *codes, float *scales, uint32_t *err_word, void *stream) {
  if (rows < 1 || cols < 1) return fail(ADC_EINVAL, "activation matrix must have at least one element");
  if (!x || !codes || !scales) return fail(ADC_EINVAL, "null buffer");
  if (!valid_float_dtype(in_dtype)) return fail(ADC_EINVAL, "activation dtype must be f32, bf16 or f16");
  if (group_size < 1) return fail(ADC_EINVAL, "group_size must be positive");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  if (launch_int8_compress(c, x, in_dtype, rows * cols, group_size, codes, scales, err_word))
    return fail(ADC_EINVAL, "int8 dispatch");
  return check_launch("int8_compress");
}

int adc_decompress_int8(const int8_t *codes, const float *scales, int64_t rows, int64_t cols,
                        int64_t group_size, void *y, int out_dtype, void *stream) {
  if (rows < 1 || cols < 1 || !codes || !scales || !y) return fail(ADC_EINVAL, "bad arguments");
  if (group_size < 1) return fail(ADC_EINVAL, "group_size must be positive");
  if (!valid_float_dtype(out_dtype)) return fail(ADC_EINVAL, "output dtype must be f32, bf16 or f16");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  if (launch_int8_decompress(c, codes, scales, rows * cols, group_size, y, out_dtype))
    return fail(ADC_EINVAL, "int8 decompress dispatch (codes need 8-byte, output 16-byte alignment)");
  return check_launch("int8_decompress");
}

int adc_compress_int4f32(const void *x, int in_dtype, int64_t rows, int64_t cols, int64_t group_size,
                         uint8_t *codes, float *scales, uint32_t *err_word, void *stream) {
  if (rows < 1 || cols < 1) return fail(ADC_EINVAL, "activation matrix must have at least one element");
  if (!x || !codes || !scales) return fail(ADC_EINVAL, "null buffer");
  if (!valid_float_dtype(in_dtype)) return fail(ADC_EINVAL, "activation dtype must be f32, bf16 or f16");
  if (group_size < 1) return fail(ADC_EINVAL, "group_size must be positive");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  if (launch_int4f32_compress(c, x, in_dtype, rows * cols, group_size, codes, scales, err_word))
    return fail(ADC_EINVAL, "int4/f32 dispatch");
  return check_launch("int4f32_compress");
}

int adc_decompress_int4f32(const uint8_t *codes, const float *scales, int64_t rows, int64_t cols,
                           int64_t group_size, void *y, int out_dtype, void *stream) {
  if (rows < 1 || cols < 1 || !codes || !scales || !y) return fail(ADC_EINVAL, "bad arguments");
  if (group_size < 1) return fail(ADC_EINVAL, "group_size must be positive");
  if (!valid_float_dtype(out_dtype)) return fail(ADC_EINVAL, "output dtype must be f32, bf16 or f16");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  if (launch_int4f32_decompress(c, codes, scales, rows * cols, group_size, y, out_dtype))
    return fail(ADC_EINVAL, "int4/f32 decompress dispatch (codes need 4-byte, output 16-byte alignment)");
  return check_launch("int4f32_decompress");
}

int adc_serialize(int scheme, const uint16_t *scales, const uint16_t *offsets, const uint8_t *codes,
                  const uint32_t *outlier_idx, const uint16_t *outlier_val, const int32_t *k_dev,
                  int64_t k_cap, int64_t rows, int64_t cols, int64_t group_size, uint8_t *out,
                  size_t out_cap, uint64_t *out_len, uint32_t *err_word, void *stream) {
  int64_t n_groups = 0, code_bytes = 0;
  if (adc_payload_bytes(scheme, rows, cols, group_size, 0, &n_groups, &code_bytes, nullptr) != ADC_OK)
    return ADC_EINVAL;
  if (rows > 0xffffffffll || cols > 0xffffffffll) return fail(ADC_EINVAL, "shape exceeds the u32 header fields");
  if (!codes || !out || !out_len) return fail(ADC_EINVAL, "null buffer");
  if (scheme != ADC_BIT_MASK && !scales) return fail(ADC_EINVAL, "null scales");
  if (scheme == ADC_ASYMMETRIC_GROUP && !offsets) return fail(ADC_EINVAL, "null offsets");
  const bool outl = scheme == ADC_OUTLIER_SEPARATED && k_cap > 0;
  if (outl && (!outlier_idx || !outlier_val || !k_dev)) return fail(ADC_EINVAL, "outlier buffers required");
  if (reinterpret_cast<uintptr_t>(out) % 16) return fail(ADC_EINVAL, "out must be 16-byte aligned");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  launch_wire_serialize(c, scheme, rows, cols, group_size, n_groups, scheme == ADC_BIT_MASK ? nullptr : scales,
                        scheme == ADC_ASYMMETRIC_GROUP ? offsets : nullptr, codes, code_bytes,
                        outl ? outlier_idx : nullptr, outl ? outlier_val : nullptr, outl ? k_dev : nullptr,
                        outl ? k_cap : 0, out, static_cast<int64_t>(out_cap), out_len, err_word);
  return check_launch("serialize");
}

int adc_parse_header(const uint8_t *header, uint64_t len, adc_wire_header *h) {
  if (!h) return ADC_WIRE_TRUNCATED;
  std::memset(h, 0, sizeof(*h));
  if (!header || len < 25) return ADC_WIRE_TRUNCATED;
  auto u32 = [&](int at) {
    uint32_t v;
    std::memcpy(&v, header + at, 4);  // little-endian host (x86-64 / aarch64)
    return v;
  };
  h->scheme = header[4];
  h->rows = u32(5), h->cols = u32(9), h->group_size = u32(13), h->group_count = u32(17),
  h->outlier_count = u32(21);
  if (std::memcmp(header, "ADC1", 4) != 0) return ADC_WIRE_BAD_MAGIC;
  if (h->scheme > ADC_BIT_MASK) return ADC_WIRE_BAD_SCHEME;
  if (h->rows < 1 || h->cols < 1) return ADC_WIRE_BAD_SHAPE;
  const uint64_t k = h->outlier_count, n = static_cast<uint64_t>(h->rows) * h->cols;
  if (h->scheme != ADC_OUTLIER_SEPARATED && k) return ADC_WIRE_OUTLIERS_NOT_ALLOWED;
  if (2 * k > h->cols) return ADC_WIRE_TOO_MANY_OUTLIERS;
  uint64_t meta = 0;
  if (h->scheme == ADC_BIT_MASK) {
    h->expected_groups = 0;
    h->code_bytes = (n + 7) / 8;
  } else {
    // u32 group_size is never negative: 0 = PER_CHANNEL (codec.py:482-487)
    h->expected_groups = h->group_size == ADC_PER_CHANNEL ? h->cols : (n + h->group_size - 1) / h->group_size;
    h->code_bytes = (n + 1) / 2;
    meta = h->expected_groups * (h->scheme == ADC_ASYMMETRIC_GROUP ? 4 : 2);
  }
  if (h->group_count != h->expected_groups) return ADC_WIRE_BAD_GROUP_COUNT;
  // n < 2^64 and k * (4 + 2 rows) < 2^63 (k < 2^31, rows < 2^32): no overflow
  h->total_bytes = 25 + meta + h->code_bytes + k * (4 + 2 * static_cast<uint64_t>(h->rows));
  if (len != h->total_bytes) return ADC_WIRE_SIZE_MISMATCH;
  return ADC_WIRE_OK;
}

int adc_deserialize(const uint8_t *in, const adc_wire_header *h, uint16_t *scales, uint16_t *offsets,
                    uint8_t *codes, uint32_t *outlier_idx, uint16_t *outlier_val, uint32_t *err_word,
                    void *stream) {
  if (!h || !in || !codes || !err_word) return fail(ADC_EINVAL, "null buffer");
  adc_wire_header chk;
  uint8_t hdr[25];
  std::memcpy(hdr, "ADC1", 4);
  hdr[4] = static_cast<uint8_t>(h->scheme);
  const uint32_t f[5] = {h->rows, h->cols, h->group_size, h->group_count, h->outlier_count};
  std::memcpy(hdr + 5, f, sizeof f);
  if (adc_parse_header(hdr, h->total_bytes, &chk) != ADC_WIRE_OK || chk.total_bytes != h->total_bytes ||
      chk.code_bytes != h->code_bytes)
    return fail(ADC_EINVAL, "header not accepted by adc_parse_header");
  const bool mask = h->scheme == ADC_BIT_MASK;
  if (!mask && !scales) return fail(ADC_EINVAL, "null scales");
  if (h->scheme == ADC_ASYMMETRIC_GROUP && !offsets) return fail(ADC_EINVAL, "null offsets");
  if (h->outlier_count && (!outlier_idx || !outlier_val)) return fail(ADC_EINVAL, "outlier buffers required");
  if (reinterpret_cast<uintptr_t>(codes) % 16) return fail(ADC_EINVAL, "codes must be 16-byte aligned");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  launch_wire_deserialize(c, in, h->scheme, h->rows, h->cols, mask ? 0 : static_cast<int64_t>(h->group_count),
                          static_cast<int64_t>(h->code_bytes), h->outlier_count, scales,
                          h->scheme == ADC_ASYMMETRIC_GROUP ? offsets : nullptr, codes, outlier_idx,
                          outlier_val, err_word);
  return check_launch("deserialize");
}

int adc_channel_abs_sums(const void *x, int in_dtype, int64_t rows, int64_t cols, double *sums,
                         uint32_t *err_word, void *workspace, size_t workspace_bytes,
                         void *stream) {
  if (rows < 1 || cols < 1 || !x || !sums) return fail(ADC_EINVAL, "bad arguments");
  if (!valid_float_dtype(in_dtype)) return fail(ADC_EINVAL, "bad dtype");
  if (!workspace || workspace_bytes < workspace_layout(cols, nullptr, nullptr))
    return fail(ADC_EWORKSPACE, "workspace too small");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  Workspace ws;
  workspace_layout(cols, &ws, workspace);
  launch_colstats_sum(c, x, in_dtype, rows, cols, ws, false, 0.0, 0, nullptr, nullptr, err_word,
                      false);
  if (cudaMemcpyAsync(sums, ws.colsum, sizeof(double) * cols, cudaMemcpyDeviceToDevice, c.stream) !=
      cudaSuccess)
    return check_launch("channel_abs_sums copy");
  return check_launch("channel_abs_sums");
}

int adc_detect_outliers(const void *x, int in_dtype, int64_t rows, int64_t cols,
                        double z_threshold, int64_t k_cap, uint32_t *outlier_idx, int32_t *k_out,
                        uint32_t *err_word, void *workspace, size_t workspace_bytes,
                        void *stream) {
  if (rows < 1 || cols < 1 || !x || !k_out) return fail(ADC_EINVAL, "bad arguments");
  if (k_cap > 0 && !outlier_idx) return fail(ADC_EINVAL, "null index buffer");
  if (!valid_float_dtype(in_dtype)) return fail(ADC_EINVAL, "bad dtype");
  if (!workspace || workspace_bytes < workspace_layout(cols, nullptr, nullptr))
    return fail(ADC_EWORKSPACE, "workspace too small");
  Ctx c{static_cast<cudaStream_t>(stream), sm_count()};
  Workspace ws;
  workspace_layout(cols, &ws, workspace);
  launch_colstats_sum(c, x, in_dtype, rows, cols, ws, true, z_threshold, k_cap, outlier_idx, k_out,
                      err_word, false);
  return check_launch("detect_outliers");
}

}  // extern "C"
