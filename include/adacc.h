/*
 * adacc.h -- C-ABI of the B200 activation-compressor path (Adacc, arXiv 2508.00806).
 *
 * This is the drop-in boundary for the reference's codec module
 * (/root/reference/pkg/src/actplan/codec.py).  Every entry point below names
 * the reference function it replaces.  Conventions:
 *
 *   - All array arguments are DEVICE pointers owned by the caller; the library
 *     never allocates.  `workspace` is caller-owned scratch of
 *     adc_workspace_bytes() bytes (256-byte aligned) that must be zero-filled
 *     once before its first use; every call leaves its counters at zero
 *     again, so a workspace is reusable by stream-ordered calls without
 *     re-clearing (the cross-CTA arrival counters live there).
 *   - Calls are stream-ordered and asynchronous on `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  Return value is a
 *     synchronous status: ADC_OK, ADC_EINVAL (argument validation, the
 *     reference's ValidationError), ADC_EWORKSPACE, or ADC_ECUDA (launch
 *     failure; adc_last_error() has the text).
 *   - Data-dependent failures are OR-ed into the device word `err_word` as
 *     ADC_ERR_* bits (never cleared by the library): non-finite after the
 *     float16 cast (NonFiniteInputError, codec.py:167-170), more than half the
 *     channels flagged (TooManyOutliersError, codec.py:324-327), k above the
 *     caller's side-buffer capacity, or a non-binary mask (NonBinaryMaskError,
 *     codec.py:355-357).  Outputs are unspecified when a bit is set.
 *   - Inputs are C-contiguous (rows, cols) matrices, channel = last dim
 *     (rows = product of the leading dims, codec.py:161-162).  Input dtypes:
 *     ADC_F32, ADC_BF16, ADC_F16 (all cast to float16 RNE first, codec.py:158);
 *     masks additionally ADC_U8 (bytes 0/1, bool tensors).
 *   - Payload layout is the reference's (codec.py:85-145): float16 scales
 *     (and offsets) as uint16 bit patterns, one per group; packed int4 codes,
 *     earlier element in the low nibble, row-major groups over the flattened
 *     tensor, COLUMN-major for group_size == ADC_PER_CHANNEL; outlier indices
 *     ascending uint32; outlier values float16 laid out (k, rows).
 *   - Reentrant: concurrent calls are safe with distinct buffers/workspaces.
 */
#ifndef ADACC_H
#define ADACC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADC_ABI_VERSION 1

#if defined(__GNUC__)
#define ADC_API __attribute__((visibility("default")))
#else
#define ADC_API
#endif

/* Scheme ids == reference Scheme IntEnum == ADC1 scheme byte (codec.py:56-60). */
#define ADC_SYMMETRIC_GROUP 0
#define ADC_ASYMMETRIC_GROUP 1
#define ADC_OUTLIER_SEPARATED 2
#define ADC_BIT_MASK 3

/* group_size sentinel: one group per channel (codec.py:45). */
#define ADC_PER_CHANNEL 0

/* element dtypes */
#define ADC_F32 0
#define ADC_BF16 1
#define ADC_F16 2
#define ADC_U8 3

/* synchronous status codes */
#define ADC_OK 0
#define ADC_EINVAL (-1)
#define ADC_ECUDA (-2)
#define ADC_EWORKSPACE (-3)

/* device error-word bits */
#define ADC_ERR_NONFINITE 1u
#define ADC_ERR_TOO_MANY_OUTLIERS 2u
#define ADC_ERR_K_CAP 4u
#define ADC_ERR_NONBINARY 8u
/* adc_deserialize content checks (CorruptPayloadError, codec.py:512-534) */
#define ADC_ERR_BAD_SCALE 16u       /* a scale is non-finite or negative */
#define ADC_ERR_BAD_OFFSET 32u      /* an offset is non-finite */
#define ADC_ERR_BAD_INDEX_RANGE 64u /* an outlier index >= cols */
#define ADC_ERR_BAD_INDEX_ORDER 128u /* outlier indices not strictly increasing */

/* adc_parse_header verdicts (CorruptPayloadError, codec.py:464-493), in the
 * reference's check order; ADC_WIRE_OK = the header describes `len` bytes. */
#define ADC_WIRE_OK 0
#define ADC_WIRE_TRUNCATED 1      /* len < 25 */
#define ADC_WIRE_BAD_MAGIC 2
#define ADC_WIRE_BAD_SCHEME 3
#define ADC_WIRE_BAD_SHAPE 4      /* rows < 1 or cols < 1 */
#define ADC_WIRE_OUTLIERS_NOT_ALLOWED 5
#define ADC_WIRE_TOO_MANY_OUTLIERS 6 /* 2k > cols */
#define ADC_WIRE_BAD_GROUP_SIZE 7
#define ADC_WIRE_BAD_GROUP_COUNT 8
#define ADC_WIRE_SIZE_MISMATCH 9

/* The 25-byte ADC1 header <4sBIIIII> (codec.py:52) and derived sizes. */
typedef struct {
  int32_t scheme;
  uint32_t rows, cols, group_size, group_count, outlier_count;
  uint64_t expected_groups; /* what the shape implies (ADC_WIRE_BAD_GROUP_COUNT) */
  uint64_t code_bytes;      /* packed codes, or mask bytes for BIT_MASK */
  uint64_t total_bytes;     /* 25 + payload (ADC_WIRE_SIZE_MISMATCH) */
} adc_wire_header;

/* Library / ABI identification. */
ADC_API const char *adc_version(void);
ADC_API int adc_abi_version(void);
/* Text of the last failing call on this host thread ("" if none). */
ADC_API const char *adc_last_error(void);
/* Number of CUDA kernels launched by this library since load (all threads). */
ADC_API unsigned long long adc_kernel_launches(void);

/*
 * Kernel-path selection (tuning / A-B testing; results are identical):
 *   "pdl"           1 = launch with programmatic dependent launch (0 default).
 *   "epl"           32 (default) or 16 elements per lane in the group
 *                   quantisers (also ADC_EPL=16).
 *   "outlier_path"  0 = column-statistics launch + quantiser launch, 1 = the
 *                   single-pass cooperative kernel wherever eligible, 2 =
 *                   automatic (default: the single pass for tall tensors of
 *                   <= 1024 columns, >= 2^25 elements, where it measured
 *                   faster).  Also ADC_OUTLIER_PATH=0/1/2.
 *   "outlier_decompress"  0 = dequantiser launch + outlier overwrite launch,
 *                   2 = one launch (output tiles dequantised into shared
 *                   memory, overwritten there, stored whole) wherever
 *                   eligible (default).
 *   "outlier_tile"  elements per tile of that launch: 4096, 8192 (default)
 *                   or 16384.
 *   "k4_trace"      1 = record the single-pass kernel's phase timestamps.
 *   "sum_smem_cols" the column-statistics tail keeps the sums in shared
 *                   memory up to this many columns (default and max 8192;
 *                   lower = smaller CTA footprint, slower tail).
 *   "cr_trace"      1 = record the column-statistics kernel's phase
 *                   timestamps instead (adc_debug_trace_k4 then returns
 *                   those: 4 u64 per CTA, the tail's at 4096 * 4).
 *   "k4_dbg"        timing experiments only (1 = stop the single pass after
 *                   its streaming phase; results invalid).
 *   "cr_rows8"      2 (default) = the column pass gives every row lane at
 *                   least 8 rows, in whole batches of 8 when a lane holds
 *                   fewer than 8 batches; 1 = at least 8 rows only; 0 = one
 *                   full wave of CTAs whatever the row count.
 *   "outlier_pdl"   1 (default) = the zeroing / per-channel quantiser is a
 *                   programmatic dependent launch of the column pass and
 *                   loads its first x units while the statistics finish;
 *                   0 = a plain stream-ordered launch.
 */
ADC_API int adc_set_option(const char *key, int value);

/*
 * Tuning aid: with adc_set_option("k4_trace", 1) the single-pass
 * outlier-separated kernel records per-CTA phase timestamps; this copies the
 * last launch's records (64 u64 per CTA: globaltimer at entry, clock64 deltas
 * at phase ends, per-warp entry / exit) to host memory.  Returns the count.
 */
ADC_API int adc_debug_trace_k4(unsigned long long *out, int n);

/*
 * Closed-form payload size; replaces packed_payload_bytes (codec.py:133-145).
 * Writes the group count, packed-code bytes and total payload bytes (any
 * output pointer may be NULL).  Host-only, no CUDA.
 */
ADC_API int adc_payload_bytes(int scheme, int64_t rows, int64_t cols, int64_t group_size,
                      int64_t outlier_count, int64_t *n_groups, int64_t *code_bytes,
                      int64_t *payload_bytes);

/* Scratch bytes adc_compress / adc_detect_outliers need for this shape. */
ADC_API size_t adc_workspace_bytes(int scheme, int64_t rows, int64_t cols, int64_t group_size);

/*
 * Compress one activation matrix; replaces compress (codec.py:381-389) and
 * thereby quantize_symmetric (:245), quantize_asymmetric (:255),
 * compress_outlier_separated (:308) and pack_bitmask (:344).
 *
 *   codes       ceil(rows*cols/2) bytes (BIT_MASK: ceil(rows*cols/8) mask bytes)
 *   scales      n_groups uint16 (f16 bits); unused for BIT_MASK
 *   offsets     n_groups uint16; ASYMMETRIC_GROUP only
 *   outlier_idx k_cap uint32, outlier_val k_cap*rows uint16, k_out one int32:
 *               OUTLIER_SEPARATED only.  k_out receives k even when k > k_cap
 *               (then ADC_ERR_K_CAP is raised and idx/val are incomplete).
 *   z_threshold OUTLIER_SEPARATED z-score threshold (codec.py:43, strict >).
 */
ADC_API int adc_compress(int scheme, const void *x, int in_dtype, int64_t rows, int64_t cols,
                 int64_t group_size, double z_threshold, int64_t k_cap,
                 uint8_t *codes, uint16_t *scales, uint16_t *offsets,
                 uint32_t *outlier_idx, uint16_t *outlier_val, int32_t *k_out,
                 uint32_t *err_word, void *workspace, size_t workspace_bytes, void *stream);

/*
 * Decompress; replaces decompress (codec.py:392-395) = dequantize (:261-286)
 * / unpack_bitmask (:372-378).  `y` is (rows, cols) of out_dtype: ADC_F32
 * reproduces the reference output bit-exactly; ADC_BF16 / ADC_F16 are the
 * float32 result rounded RNE (training mode).  BIT_MASK writes 0/1 bytes
 * (out_dtype ADC_U8).  `k_dev` is the device outlier count written by
 * adc_compress; at most k_cap outlier columns are scattered.
 */
ADC_API int adc_decompress(int scheme, const uint8_t *codes, const uint16_t *scales,
                   const uint16_t *offsets, const uint32_t *outlier_idx,
                   const uint16_t *outlier_val, const int32_t *k_dev, int64_t k_cap,
                   int64_t rows, int64_t cols, int64_t group_size, void *y, int out_dtype,
                   void *stream);

/*
 * EXTENSION, no reference counterpart (north_star names int8 codes with fp32
 * scales; the reference has only int4): symmetric group int8.
 * Parity unpinned -- semantics defined by this library and restated in
 * oracle/int8_oracle.py: h = f16(x); per group of group_size row-major
 * elements s = f32(max|h| / 127); code = clip(rint_even(f32(h / s)), -127,
 * 127) (s = 0 divides by 1); decompress = f32(code * s) (then RNE to the
 * output dtype).  codes: rows*cols int8; scales: ceil(rows*cols/group) f32.
 * Non-finite inputs raise ADC_ERR_NONFINITE in err_word.
 */
ADC_API int adc_compress_int8(const void *x, int in_dtype, int64_t rows, int64_t cols,
                              int64_t group_size, int8_t *codes, float *scales, uint32_t *err_word,
                              void *stream);
ADC_API int adc_decompress_int8(const int8_t *codes, const float *scales, int64_t rows, int64_t cols,
                                int64_t group_size, void *y, int out_dtype, void *stream);

/*
 * EXTENSION, no reference counterpart (north_star "fp32-scale storage
 * option"; the reference rounds every scale to float16, codec.py:192-196):
 * the symmetric group int4 codec with FLOAT32 scales.  Parity unpinned,
 * restated in oracle/int8_oracle.py: h = f16(x); s = f32(max|h| / 8) per
 * group of group_size row-major elements; code = clip(rint_even(f32(h / s')),
 * -8, 7) (s' = 1 for an all-zero group), nibbles packed as the reference's
 * (codec.py:199-203); decompress = f32(code * s) (then RNE to the output
 * dtype).  codes: ceil(rows*cols/2) bytes; scales: ceil(rows*cols/group) f32.
 */
ADC_API int adc_compress_int4f32(const void *x, int in_dtype, int64_t rows, int64_t cols,
                                 int64_t group_size, uint8_t *codes, float *scales, uint32_t *err_word,
                                 void *stream);
ADC_API int adc_decompress_int4f32(const uint8_t *codes, const float *scales, int64_t rows, int64_t cols,
                                   int64_t group_size, void *y, int out_dtype, void *stream);

/*
 * Device-side ADC1 wire format; replaces serialize (codec.py:432-459) without
 * a host round trip: writes the 25-byte header, metadata, codes and outlier
 * side buffer of a compressed tensor (the device buffers adc_compress wrote)
 * into `out` (16-byte aligned device memory, out_cap bytes) and the total
 * length into the device word *out_len.  If the payload exceeds out_cap it
 * is truncated and ADC_ERR_K_CAP is raised in err_word.
 */
ADC_API int adc_serialize(int scheme, const uint16_t *scales, const uint16_t *offsets,
                          const uint8_t *codes, const uint32_t *outlier_idx,
                          const uint16_t *outlier_val, const int32_t *k_dev, int64_t k_cap,
                          int64_t rows, int64_t cols, int64_t group_size, uint8_t *out,
                          size_t out_cap, uint64_t *out_len, uint32_t *err_word, void *stream);

/*
 * ADC1 header check; the header half of deserialize (codec.py:464-493).
 * Host-only, no CUDA: reads the first 25 bytes of a HOST copy of the header,
 * fills *h and returns an ADC_WIRE_* verdict (the first failing check in the
 * reference's order); `len` is the whole payload's length in bytes.
 */
ADC_API int adc_parse_header(const uint8_t *header, uint64_t len, adc_wire_header *h);

/*
 * Device-side ADC1 deserialisation; the content half of deserialize
 * (codec.py:494-546).  `in` is the whole payload in DEVICE memory, `h` its
 * header as accepted by adc_parse_header (ADC_WIRE_OK, else ADC_EINVAL).
 * Splits the payload into the record's device arrays -- scales (and offsets)
 * h->group_count uint16 each, codes h->code_bytes (16-byte aligned), outlier
 * indices k uint32 and values k*rows uint16 -- and ORs ADC_ERR_BAD_* bits into
 * err_word for non-finite / negative scales, non-finite offsets, indices
 * >= cols and indices that do not strictly increase.  BIT_MASK: `codes`
 * receives the mask bytes.
 */
ADC_API int adc_deserialize(const uint8_t *in, const adc_wire_header *h, uint16_t *scales,
                            uint16_t *offsets, uint8_t *codes, uint32_t *outlier_idx,
                            uint16_t *outlier_val, uint32_t *err_word, void *stream);

/* Column sums of |f16(x)| in float64; replaces channel_abs_sums (codec.py:289-291). */
ADC_API int adc_channel_abs_sums(const void *x, int in_dtype, int64_t rows, int64_t cols,
                         double *sums, uint32_t *err_word, void *workspace,
                         size_t workspace_bytes, void *stream);

/*
 * Outlier channel indices; replaces detect_outlier_channels (codec.py:294-305).
 * Writes ascending indices (up to k_cap) and k.
 */
ADC_API int adc_detect_outliers(const void *x, int in_dtype, int64_t rows, int64_t cols,
                        double z_threshold, int64_t k_cap, uint32_t *outlier_idx,
                        int32_t *k_out, uint32_t *err_word, void *workspace,
                        size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ADACC_H */
