// K4 detection half: exact channel |x|-sums and the numpy-identical z-score,
// plus the per-channel abs-max pass of K3 -- one kernel launch each.
//
// Reference: channel_abs_sums (codec.py:289-291), detect_outlier_channels
// (:294-305), the TooManyOutliers guard and index layout of
// compress_outlier_separated (:321-341); per-channel scales (:181-182, 225-227).
//
// One launch, two stages, chained with the last-block-done pattern:
//   A. a full wave of CTAs (grid = column strips x row blocks sized to the
//      SM count and the measured occupancy) streams the matrix once with
//      8 x 128-bit loads in flight per thread (L2 evict_last, so the
//      quantisation pass that follows re-reads from L2 when it fits), folds
//      its 8 row lanes in shared memory and adds its 256 column partials
//      into global accumulators with f64 atomics (sum) / u32 atomicMax (max);
//   B. the last CTA to arrive moves the accumulators to the outputs, resets
//      them, and computes mean / std / z / flags / ranks (stats.cuh).
// Accumulators and counters are reset by the CTA that consumes them, so the
// workspace stays zero-filled between calls (the caller zero-fills it once).
//
// Exactness: every f16 value is an integer multiple
// of 2^-24 below 2^16, so every float64 partial sum -- thread, CTA, atomic --
// is exact, hence independent of order, while the column total is < 2^29.
// Round-to-nearest is monotone, so a total that reaches 2^29 is seen as
// >= 2^29 whatever the order; then the final CTA recomputes every column in
// numpy's row order.  The mean / std use numpy's pairwise summation tree
// (block 128, unroll 8, initial 0.0; restated in
// oracle/codec_oracle.py:pairwise_sum and pinned against ndarray.sum); every
// float64 op is an explicit _rn intrinsic so nothing is contracted into an FMA.
#include "common.cuh"
#include "launch.h"
#include "quant.cuh"
#include "stats.cuh"

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdlib>

namespace adc {

constexpr double kExactLimit = 536870912.0;  // 2^29
constexpr int kStripCols = 256;              // 32 column units of 8 per CTA
constexpr int kRowLanes = kThreads / 32;     // 8
constexpr int kSmemSumCols = 8192;           // the final CTA keeps S in shared memory up to here (max)
static int g_sum_smem_cols = kSmemSumCols;   // tuning: "sum_smem_cols" lowers it
// tuning "cr_rows8" (1, the default): at least 8 rows per row lane, so a
// short matrix runs whole batches of 8 loads in flight on fewer CTAs instead
// of a full wave whose warps fetch their few rows one dependent load at a
// time.  Same box: [8192,1024] column sums 10.2 -> 9.0 us, outlier-separated
// compress 19.5 -> 18.4 us, per-channel 10.8 -> 10.0 us, bench step 4775 ->
// 4814 GB/s; taller matrices keep the full wave (unchanged).
// Mode 2 (the default) also shrinks the wave of a matrix with fewer than 8
// batches per row lane until every lane's rows are whole batches of 8 (keeping
// at least half the wave): [8192,4096] 37 -> 32 row blocks.  Same box, against
// mode 1: [8192,4096] per-channel 31.1 -> 30.2 us, outlier-separated 48.5 ->
// 48.1 us (two boxes), bench step 4738 -> 4843 GB/s on one box, a tie on the
// other; applied to [131072,1024] it measured slower (column sums 46.5 ->
// 50.3 us), hence the 8-batch bound.
static int g_cr_rows8 = 2;
constexpr int kStageASmem = kRowLanes * 32 * 8 * sizeof(double);
// dynamic shared memory of a launch: the stage A fold buffer, or (sum mode,
// cols <= kSmemSumCols) the column sums + the statistics scratch for the tail
// (exact: rounding it up to 8 KB buckets measured 3% slower on the
// 4-stream bench step -- larger footprints co-reside less with the other
// streams' kernels; the occupancy cache below holds 32 sizes, beyond that the
// query simply runs per call)
constexpr int kMaxColSmem = ((kSmemSumCols * 8 + 15) & ~15) + kStatsScratch;
static_assert(kMaxColSmem >= kStageASmem, "attribute covers the stage A buffer");
static inline int col_smem(bool sum, int64_t cols) {
  const int64_t tail = (sum && cols <= g_sum_smem_cols) ? ((cols * 8 + 15) & ~int64_t{15}) + kStatsScratch : 0;
  return static_cast<int>(tail > kStageASmem ? tail : (kStageASmem > kStatsScratch ? kStageASmem : kStatsScratch));
}

// f16 half of a packed word -> f64 in one F2F.F64.F16 (reads .H0/.H1 directly;
// keeps the integer pipe free -- the bit-trick version was ALU-bound).
__device__ __forceinline__ double h_lo_f64(uint32_t w) {
  double r;
  asm("cvt.f64.f16 %0, %1;" : "=d"(r) : "h"(static_cast<unsigned short>(w & 0xffffu)));
  return r;
}
__device__ __forceinline__ double h_hi_f64(uint32_t w) {
  double r;
  asm("cvt.f64.f16 %0, %1;" : "=d"(r) : "h"(static_cast<unsigned short>(w >> 16)));
  return r;
}

struct ColArgs {
  int64_t rows, cols;
  double *acc;          // [cols] f64 sum accumulators, zero at rest
  uint32_t *macc;       // [cols] u32 max accumulators, zero at rest
  double *S;            // column sums (sum mode)
  uint32_t *colmax;     // column abs-max f16 bits (max mode)
  uint32_t *done_cnt;   // [0] CTAs finished
  // stats (sum mode)
  int do_stats, too_many_check;
  double thr;
  int64_t k_cap;
  int trace;  // record phase timestamps (tuning, "cr_trace")
  int64_t smem_cols;  // S stays in shared memory up to this many columns
  Tree tree;
  uint8_t *flag;
  uint32_t *idx;
  int32_t *k_out;
  uint32_t *err;
};

// Phase timestamps of the last traced launch (tuning): per CTA [0] entry,
// [1] stage A done, [2] arrival; then at kCrTraceCtas * 4: the last CTA's
// [0] tail start, [1] accumulators moved, [2] statistics done.
constexpr int kCrTraceCtas = 4096;
__device__ unsigned long long g_crtrace[kCrTraceCtas * 4 + 16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CR_TRACE(slot)                                                                         \
  do {                                                                                         \
    const int cta_ = blockIdx.y * gridDim.x + blockIdx.x;                                      \
    if (a.trace && threadIdx.x == 0 && cta_ < kCrTraceCtas) g_crtrace[cta_ * 4 + (slot)] = gtimer(); \
  } while (0)
#define CR_TRACE_TAIL(slot)                                                                    \
  do {                                                                                         \
    if (a.trace && threadIdx.x == 0) g_crtrace[kCrTraceCtas * 4 + (slot)] = gtimer();          \
  } while (0)

// numpy's row-order float64 column sums (only when some total >= 2^29)
template <int DT>
__device__ void numpy_order_sums(const void *x, int64_t rows, int64_t cols, double *S) {
  for (int64_t cc = threadIdx.x; cc < cols; cc += blockDim.x) {
    double s = 0.0;
    for (int64_t r = 0; r < rows; ++r)
      s = __dadd_rn(s, fabs(static_cast<double>(h2f(Loader<DT>::load1(x, r * cols + cc)))));
    __stcg(S + cc, s);
  }
}

template <int DT, bool SUM>
__global__ void __launch_bounds__(kThreads, 4) colreduce(const void *__restrict__ x, ColArgs a) {
  pdl_wait();  // dependents are triggered after the arrival below, not here
  // stage A reduction buffer; the last CTA reuses it for S and the stats scratch
  extern __shared__ __align__(16) unsigned char s_buf[];  // col_smem(SUM, cols) bytes
  double(*red)[32][8] = reinterpret_cast<double(*)[32][8]>(s_buf);
  __shared__ int s_last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t cols = a.cols, rows = a.rows;
  const int64_t cu = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  const bool live = cu * 8 < cols;
  CR_TRACE(0);

  // ---- stage A: this CTA's rows, 8 columns per thread, 8 loads in flight
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t mx[4] = {0, 0, 0, 0};
  if (live) {
    const int64_t step = static_cast<int64_t>(gridDim.y) * kRowLanes;
    int64_t r = static_cast<int64_t>(blockIdx.y) * kRowLanes + ty;
    for (; r + 7 * step < rows; r += 8 * step) {
      uint4 h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = Loader<DT>::template load8<true>(x, (r + q * step) * cols + cu * 8);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t w[4] = {h[q].x, h[q].y, h[q].z, h[q].w};
        if (SUM) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[2 * j] = __dadd_rn(acc[2 * j], fabs(h_lo_f64(w[j])));
            acc[2 * j + 1] = __dadd_rn(acc[2 * j + 1], fabs(h_hi_f64(w[j])));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) mx[j] = __vmaxu2(mx[j], w[j] & 0x7fff7fffu);
        }
      }
    }
    for (; r < rows; r += step) {
      const uint4 h = Loader<DT>::template load8<true>(x, r * cols + cu * 8);
      const uint32_t w[4] = {h.x, h.y, h.z, h.w};
      if (SUM) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[2 * j] = __dadd_rn(acc[2 * j], fabs(h_lo_f64(w[j])));
          acc[2 * j + 1] = __dadd_rn(acc[2 * j + 1], fabs(h_hi_f64(w[j])));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) mx[j] = __vmaxu2(mx[j], w[j] & 0x7fff7fffu);
      }
    }
  }
  CR_TRACE(1);
  if (SUM) {
#pragma unroll
    for (int j = 0; j < 8; ++j) red[ty][tx][j] = acc[j];
  } else {
    uint32_t *redu = reinterpret_cast<uint32_t *>(&red[0][0][0]);
#pragma unroll
    for (int j = 0; j < 4; ++j) redu[(ty * 32 + tx) * 4 + j] = mx[j];
  }
  __syncthreads();
  // this CTA's partial of strip column t = 8*ctx + cj: fold the 8 row lanes,
  // then one atomic per column
  {
    const int t = threadIdx.x, ctx = t >> 3, cj = t & 7;
    const int64_t c = static_cast<int64_t>(blockIdx.x) * kStripCols + t;
    if (SUM) {
      double v = red[0][ctx][cj];
#pragma unroll
      for (int q = 1; q < kRowLanes; ++q) v = __dadd_rn(v, red[q][ctx][cj]);
      if (c < cols && v != 0.0) atomicAdd(a.acc + c, v);
    } else {
      const uint32_t *redu = reinterpret_cast<const uint32_t *>(&red[0][0][0]);
      uint32_t v = 0;
#pragma unroll
      for (int q = 0; q < kRowLanes; ++q) v = max(v, (redu[(q * 32 + ctx) * 4 + (cj >> 1)] >> (16 * (cj & 1))) & 0xffffu);
      if (c < cols && v != 0u) atomicMax(a.macc + c, v);
    }
  }
  // ---- stage B: the last CTA finalises.  Arrival: CTA barrier, then one
  // acq_rel atomic by thread 0 -- release publishes every thread's column
  // atomics (barrier + cumulative release, the split-K semaphore pattern),
  // acquire lets the last CTA (after its barrier) read all of them; no
  // per-thread fence
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = atom_add_acq_rel_gpu(a.done_cnt, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  CR_TRACE(2);
  // every CTA has added its partials: the zeroing quantiser (a programmatic
  // dependent) may start loading x while the last CTA finishes the statistics
  pdl_trigger();
  if (!s_last) return;
  CR_TRACE_TAIL(0);
  // move the accumulators out (8 columns per thread per round trip) and reset them
  const bool s_smem = SUM && cols <= a.smem_cols;
  double *s_S = reinterpret_cast<double *>(s_buf);
  int flagged = 0;
  for (int64_t base = 0; base < cols; base += 8 * kThreads) {
    if (SUM) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t c = base + q * kThreads + threadIdx.x;
        v[q] = c < cols ? __ldcg(a.acc + c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t c = base + q * kThreads + threadIdx.x;
        if (c < cols) {
          __stcg(a.acc + c, 0.0);
          __stcg(a.S + c, v[q]);
          if (s_smem) s_S[c] = v[q];
          flagged |= !(v[q] < kExactLimit);
        }
      }
    } else {
      uint32_t m[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t c = base + q * kThreads + threadIdx.x;
        m[q] = c < cols ? __ldcg(a.macc + c) : 0u;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t c = base + q * kThreads + threadIdx.x;
        if (c < cols) {
          __stcg(a.macc + c, 0u);
          __stcg(a.colmax + c, m[q]);
          flagged |= m[q] >= 0x7c00u;
        }
      }
    }
  }
  if (threadIdx.x == 0) a.done_cnt[0] = 0;  // reset for the next call
  flagged = __syncthreads_or(flagged);
  CR_TRACE_TAIL(1);
  if (!SUM) {
    if (flagged && threadIdx.x == 0 && a.err) atomicOr(a.err, ADC_ERR_NONFINITE);
    return;
  }
  if (flagged) {  // some total >= 2^29: numpy's row order
    numpy_order_sums<DT>(x, rows, cols, a.S);
    __syncthreads();
    if (s_smem)
      for (int64_t c = threadIdx.x; c < cols; c += kThreads) s_S[c] = __ldcg(a.S + c);
    __syncthreads();
  }
  if (a.do_stats) {
    if (s_smem)
      outlier_stats_block<true>(s_S, rows, cols, a.thr, a.k_cap, a.tree, a.flag, a.idx, a.k_out,
                                a.err, a.too_many_check != 0, s_buf + ((cols * 8 + 15) & ~int64_t{15}),
                                a.trace ? g_crtrace + kCrTraceCtas * 4 + 4 : nullptr);
    else
      outlier_stats_block<false>(a.S, rows, cols, a.thr, a.k_cap, a.tree, a.flag, a.idx, a.k_out,
                                 a.err, a.too_many_check != 0, s_buf,
                                 a.trace ? g_crtrace + kCrTraceCtas * 4 + 4 : nullptr);
  }
  CR_TRACE_TAIL(2);
}

// ---------------------------------------------------------------------------
// generic path for unaligned / cols % 8 != 0 matrices: one thread per column
// accumulates in row order (always numpy-exact), then the same stats block.
// ---------------------------------------------------------------------------
template <int DT, bool SUM>
__global__ void __launch_bounds__(kThreads) colstats_generic(const void *__restrict__ x, ColArgs a) {
  pdl_entry();
  __shared__ __align__(16) unsigned char s_raw[kStatsScratch];
  __shared__ int s_last;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; c < a.cols;
       c += static_cast<int64_t>(gridDim.x) * kThreads) {
    if (SUM) {
      double s = 0.0;
      for (int64_t r = 0; r < a.rows; ++r)
        s = __dadd_rn(s, fabs(static_cast<double>(h2f(Loader<DT>::load1(x, r * a.cols + c)))));
      __stcg(a.S + c, s);
    } else {
      uint32_t m = 0;
      for (int64_t r = 0; r < a.rows; ++r) m = max(m, Loader<DT>::load1(x, r * a.cols + c) & 0x7fffu);
      __stcg(a.colmax + c, m);
      if (m >= 0x7c00u && a.err) atomicOr(a.err, ADC_ERR_NONFINITE);
    }
  }
  if (!SUM) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.done_cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) a.done_cnt[0] = 0;
  __syncthreads();
  if (a.do_stats)
    outlier_stats_block<false>(a.S, a.rows, a.cols, a.thr, a.k_cap, a.tree, a.flag, a.idx,
                        a.k_out, a.err, a.too_many_check != 0, s_raw);
}

// ---------------------------------------------------------------------------
#define ADC_DT_SWITCH(dt, DT, ...)                                   \
  switch (dt) {                                                      \
    case ADC_F32: { constexpr int DT = ADC_F32; __VA_ARGS__; break; }  \
    case ADC_BF16: { constexpr int DT = ADC_BF16; __VA_ARGS__; break; } \
    case ADC_F16: { constexpr int DT = ADC_F16; __VA_ARGS__; break; }  \
    default: return -1;                                              \
  }

static std::atomic<int> g_cr_trace{0};
void set_cr_trace(int v) { g_cr_trace.store(v, std::memory_order_relaxed); }
void set_cr_rows8(int v) { g_cr_rows8 = v == 2 ? 2 : (v ? 1 : 0); }
void set_sum_smem_cols(int v) { g_sum_smem_cols = v < 0 ? 0 : (v > kSmemSumCols ? kSmemSumCols : v); }
int read_cr_trace(unsigned long long *host, int n) {
  n = n < kCrTraceCtas * 4 + 16 ? n : kCrTraceCtas * 4 + 16;
  return cudaMemcpyFromSymbol(host, g_crtrace, sizeof(unsigned long long) * n) == cudaSuccess ? n : -1;
}

static ColArgs make_args(int64_t rows, int64_t cols, const Workspace &ws) {
  ColArgs a{};
  a.trace = g_cr_trace.load(std::memory_order_relaxed);
  a.smem_cols = g_sum_smem_cols;
  a.rows = rows;
  a.cols = cols;
  a.acc = ws.acc;
  a.macc = ws.macc;
  a.S = ws.colsum;
  a.colmax = ws.colmax;
  a.done_cnt = ws.counters;
  a.tree = Tree{ws.node_lo, ws.node_n, ws.node_left, ws.node_val};
  a.flag = ws.flag;
  return a;
}

static bool fast_cols(const void *x, int64_t cols) {
  return cols % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
}

// One full wave: column strips x row blocks ~= SMs x resident CTAs per SM,
// at least one row per row lane.
template <typename K>
static dim3 col_grid(const Ctx &c, K kernel, int64_t rows, int64_t cols, int smem) {
  // occupancy per (kernel, dynamic shared-memory size); every instantiation
  // shares this function's type, so the cache is keyed by the kernel pointer
  struct Entry { const void *k; int smem, occ; };
  static Entry cache[32];
  static int used = 0;
  static std::mutex mu;
  int occ = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    bool seen = false;
    for (int i = 0; i < used; ++i) {
      if (cache[i].k != reinterpret_cast<const void *>(kernel)) continue;
      seen = true;
      if (cache[i].smem == smem) occ = cache[i].occ;
    }
    if (!seen)
      // the largest size any launch may request (independent of the runtime
      // sum_smem_cols setting: a smaller attribute would reject later launches)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxColSmem);
    if (occ == 0) {
      int v = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, kThreads, smem);
      occ = v > 0 ? v : 1;
      if (used < 32) cache[used++] = Entry{reinterpret_cast<const void *>(kernel), smem, occ};
    }
  }
  const int64_t gx = (cols + kStripCols - 1) / kStripCols;
  int64_t gy = static_cast<int64_t>(c.num_sms) * occ / gx;  // never a partial second wave
  // "cr_rows8": at least 8 rows per row lane, so stage A runs whole batches of 8 loads in flight
  const int64_t maxy = g_cr_rows8 ? std::max<int64_t>(1, rows / (8 * kRowLanes)) : (rows + kRowLanes - 1) / kRowLanes;
  if (g_cr_rows8 == 2 && gy > 1 && rows < 64 * kRowLanes * gy) {
    // fewer than 8 batches per row lane: make them whole -- the largest gy <= the wave with
    // rows % (8 row lanes * 8 * gy) == 0, if it keeps at least half the wave (taller matrices
    // keep the wave: there the remainder is a small share, and fewer CTAs measured slower)
    for (int64_t y = std::min(gy, maxy); y >= (gy + 1) / 2 && y >= 1; --y)
      if (rows % (8 * kRowLanes * y) == 0) {
        gy = y;
        break;
      }
  }
  if (gy > maxy) gy = maxy;
  if (gy < 1) gy = 1;
  if (gy > 65535) gy = 65535;
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
}

int launch_colstats_sum(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                        const Workspace &ws, bool do_stats, double thr, int64_t k_cap,
                        uint32_t *idx, int32_t *k_out, uint32_t *err, bool too_many_check) {
  ColArgs a = make_args(rows, cols, ws);
  a.do_stats = do_stats ? 1 : 0;
  a.too_many_check = too_many_check ? 1 : 0;
  a.thr = thr;
  a.k_cap = k_cap;
  a.idx = idx;
  a.k_out = k_out;
  a.err = err;
  if (fast_cols(x, cols)) {
    ADC_DT_SWITCH(dt, DT, {
      const int smem = col_smem(true, cols);
      const dim3 g = col_grid(c, colreduce<DT, true>, rows, cols, smem);
      launch_k(colreduce<DT, true>, g, kThreads, smem, c.stream, x, a);
      note_launches(1);
    });
  } else {
    const int g = static_cast<int>((cols + kThreads - 1) / kThreads);
    ADC_DT_SWITCH(dt, DT, (launch_k(colstats_generic<DT, true>, g, kThreads, 0, c.stream, x, a), note_launches(1)));
  }
  return 0;
}

int launch_colstats_max(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                        const Workspace &ws, uint32_t *err) {
  ColArgs a = make_args(rows, cols, ws);
  a.err = err;
  if (fast_cols(x, cols)) {
    ADC_DT_SWITCH(dt, DT, {
      const int smem = col_smem(false, cols);
      const dim3 g = col_grid(c, colreduce<DT, false>, rows, cols, smem);
      launch_k(colreduce<DT, false>, g, kThreads, smem, c.stream, x, a);
      note_launches(1);
    });
  } else {
    const int g = static_cast<int>((cols + kThreads - 1) / kThreads);
    ADC_DT_SWITCH(dt, DT, (launch_k(colstats_generic<DT, false>, g, kThreads, 0, c.stream, x, a), note_launches(1)));
  }
  return 0;
}

}  // namespace adc
