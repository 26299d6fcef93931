// K4 detection half: exact channel |x|-sums and the numpy-identical z-score,
// plus the per-channel abs-max pass of K3 -- one kernel launch each.
//
// Reference: channel_abs_sums (codec.py:289-291), detect_outlier_channels
// (:294-305), the TooManyOutliers guard and index layout of
// compress_outlier_separated (:321-341); per-channel scales (:181-182, 225-227).
//
// One launch, three stages, chained with the last-block-done pattern (no grid
// barrier, no cooperative launch, no global atomics on data):
//   A. every CTA reduces a (rows/gy) x 256-column tile into per-CTA column
//      partials, written to the workspace;
//   B. the last CTA to finish in a column strip sums that strip's partials;
//   C. the last strip to finish computes mean / std / z / flags / ranks.
// Counters are reset by the CTAs that consume them, so the workspace stays
// zero-filled between calls (it must be zero-filled once by the caller).
//
// Exactness: every f16 value is an integer multiple
// of 2^-24 below 2^16, so float64 partial sums are exact -- hence independent
// of summation order -- while the column total is < 2^29.  If any total
// reaches 2^29 the final CTA recomputes every column in numpy's row order.
// The mean / std use numpy's pairwise summation tree (block 128, unroll 8,
// initial 0.0; restated in oracle/codec_oracle.py:pairwise_sum and pinned
// against ndarray.sum), evaluated level-parallel here; every float64 op is an
// explicit _rn intrinsic so nothing is contracted into an FMA.
#include "common.cuh"
#include "launch.h"

namespace adc {

constexpr double kExactLimit = 536870912.0;  // 2^29
constexpr int kStripCols = 256;              // 32 column units of 8 per CTA

// |f16| -> f64 without the conversion pipe: f16 -> f32 (HADD2.F32), then
// re-bias the f32 exponent into an f64 (every f16 value is a normal f32).
__device__ __forceinline__ double absh_to_f64(uint32_t bits) {
  const uint32_t u = __float_as_uint(h2f(bits & 0x7fffu));
  const uint32_t hi = u ? (u >> 3) + (896u << 20) : 0u;
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
}

// ---------------------------------------------------------------------------
// block primitives (256 threads)
// ---------------------------------------------------------------------------
// Exclusive scan of v over the block; *total receives the block sum.
__device__ __forceinline__ int block_excl_scan(int v, int *total, int *s_tmp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_tmp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nw ? s_tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    if (lane < nw) s_tmp[lane] = w;
  }
  __syncthreads();
  const int before = (wid ? s_tmp[wid - 1] : 0) + incl - v;
  *total = s_tmp[nw - 1];
  __syncthreads();
  return before;
}

struct Term {  // element i of the summed vector: S[i] or (S[i]-mean)^2
  const double *s;
  double mean;
  bool squared;
  __device__ __forceinline__ double operator()(int64_t i) const {
    const double v = __ldcg(s + i);
    if (!squared) return v;
    const double d = __dsub_rn(v, mean);
    return __dmul_rn(d, d);
  }
};

// One leaf of pairwise_sum_DOUBLE computed by an aligned group of 8 lanes:
// lane j owns accumulator r[j]; the final ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// is built with width-8 shuffles in exactly that order; lane 0 adds the
// n % 8 remainder sequentially.  All 32 lanes must call it.
__device__ __forceinline__ double leaf_sum8(const Term &t, int64_t lo, int64_t n, bool valid) {
  const int j = threadIdx.x & 7;
  double res = 0.0;
  if (valid && n >= 8) {
    double r = t(lo + j);
    const int64_t stop = n - (n % 8);
    for (int64_t i = 8; i < stop; i += 8) r = __dadd_rn(r, t(lo + i + j));
    res = r;
  }
  const double a = __dadd_rn(res, __shfl_down_sync(0xffffffffu, res, 1, 8));
  const double b = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, 2, 8));
  double c = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, 4, 8));
  if (valid && j == 0) {
    if (n < 8) {
      c = 0.0;
      for (int64_t i = 0; i < n; ++i) c = __dadd_rn(c, t(lo + i));
    } else {
      for (int64_t i = n - (n % 8); i < n; ++i) c = __dadd_rn(c, t(lo + i));
    }
  }
  return c;
}

// Level-parallel evaluation of numpy's pairwise recursion over n values.
// nodes: lo/n/left/val arrays in the workspace; s_lvl: level offsets (smem).
struct Tree {
  int64_t *lo, *n;
  int32_t *left;
  double *val;
};

__device__ int build_tree(int64_t n, const Tree &tr, int *s_lvl, int *s_tmp) {
  if (threadIdx.x == 0) {
    tr.lo[0] = 0;
    tr.n[0] = n;
    s_lvl[0] = 0;
    s_lvl[1] = 1;
  }
  __syncthreads();
  int d = 0;
  for (;; ++d) {
    const int b = s_lvl[d], e = s_lvl[d + 1];
    if (b == e) break;
    int next = e;
    for (int base = b; base < e; base += blockDim.x) {
      const int i = base + threadIdx.x;
      const int64_t m = i < e ? tr.n[i] : 0;
      const int internal = (i < e && m > 128) ? 1 : 0;
      int total;
      const int before = block_excl_scan(internal, &total, s_tmp);
      if (i < e) {
        if (internal) {
          const int l = next + 2 * before;
          const int64_t lo = tr.lo[i];
          int64_t h = m / 2;
          h -= h % 8;
          tr.left[i] = l;
          tr.lo[l] = lo;
          tr.n[l] = h;
          tr.lo[l + 1] = lo + h;
          tr.n[l + 1] = m - h;
        } else {
          tr.left[i] = -1;
        }
      }
      next += 2 * total;
    }
    if (threadIdx.x == 0) s_lvl[d + 2] = next;
    __syncthreads();
  }
  return d;  // number of non-empty levels
}

__device__ double tree_sum(const Term &t, const Tree &tr, int depth, const int *s_lvl) {
  const int total_nodes = s_lvl[depth];
  const int groups = blockDim.x / 8;
  const int g = threadIdx.x / 8;
  for (int base = 0; base < total_nodes; base += groups) {
    const int i = base + g;
    const bool valid = i < total_nodes && tr.left[i] < 0;
    const double v = leaf_sum8(t, valid ? tr.lo[i] : 0, valid ? tr.n[i] : 0, valid);
    if (valid && (threadIdx.x & 7) == 0) tr.val[i] = v;
  }
  __syncthreads();
  for (int d = depth - 2; d >= 0; --d) {
    for (int i = s_lvl[d] + threadIdx.x; i < s_lvl[d + 1]; i += blockDim.x) {
      const int l = tr.left[i];
      if (l >= 0) tr.val[i] = __dadd_rn(tr.val[l], tr.val[l + 1]);
    }
    __syncthreads();
  }
  return __dadd_rn(0.0, tr.val[0]);
}

// Stage C: mean / std / z-score flags / ranks / indices (codec.py:294-305, 324-341).
__device__ void outlier_stats_block(const double *S, int64_t rows, int64_t cols, double thr,
                                    int64_t k_cap, const Tree &tr, uint8_t *flag, int32_t *rank,
                                    uint32_t *idx, int32_t *k_out, uint32_t *err,
                                    bool too_many_check) {
  __shared__ int s_lvl[72];
  __shared__ int s_tmp[32];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const double cap = 65504.0 * static_cast<double>(rows);
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
    if (!(__ldcg(S + c) <= cap)) s_bad = 1;  // inf/NaN input (no finite f16 matrix reaches it)
  const int depth = build_tree(cols, tr, s_lvl, s_tmp);
  Term t{S, 0.0, false};
  const double mean = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
  __syncthreads();
  t.mean = mean;
  t.squared = true;
  const double var = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
  const double sigma = __dsqrt_rn(var);
  int64_t pos = 0;
  for (int64_t base = 0; base < cols; base += blockDim.x) {
    const int64_t c = base + threadIdx.x;
    int f = 0;
    if (c < cols && sigma != 0.0)
      f = __ddiv_rn(__dsub_rn(__ldcg(S + c), mean), sigma) > thr ? 1 : 0;
    int total;
    const int before = block_excl_scan(f, &total, s_tmp);
    if (c < cols) {
      flag[c] = static_cast<uint8_t>(f);
      const int64_t r = pos + before;
      rank[c] = f ? static_cast<int32_t>(r) : -1;
      if (f && r < k_cap) idx[r] = static_cast<uint32_t>(c);
    }
    pos += total;
  }
  if (threadIdx.x == 0) {
    *k_out = static_cast<int32_t>(pos);
    if (err) {
      if (s_bad) atomicOr(err, ADC_ERR_NONFINITE);
      if (too_many_check && 2 * pos > cols) atomicOr(err, ADC_ERR_TOO_MANY_OUTLIERS);
      if (pos > k_cap) atomicOr(err, ADC_ERR_K_CAP);
    }
  }
}

// ---------------------------------------------------------------------------
// the single-launch column-statistics kernel
// ---------------------------------------------------------------------------
struct ColArgs {
  int64_t rows, cols;
  double *partial;      // [gy][cols] f64 (sum) or u32 (max) partials
  double *S;            // column sums (sum mode)
  uint32_t *colmax;     // column abs-max f16 bits (max mode)
  uint32_t *strip_cnt;  // [gx] arrival counters
  uint32_t *done_cnt;   // [0] strips finished, [1] inexact flag
  // stats (sum mode)
  int do_stats, too_many_check;
  double thr;
  int64_t k_cap;
  Tree tree;
  uint8_t *flag;
  int32_t *rank;
  uint32_t *idx;
  int32_t *k_out;
  uint32_t *err;
};

template <int DT, bool SUM>
__global__ void __launch_bounds__(kThreads) colstats(const void *__restrict__ x, ColArgs a) {
  __shared__ double red[8][32][8];
  __shared__ int s_last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t cols = a.cols, rows = a.rows;
  const int64_t cu = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  const bool live = cu * 8 < cols;
  const int gy = gridDim.y;

  // ---- stage A: this CTA's rows, 8 columns per thread, 4 loads in flight
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t mx[4] = {0, 0, 0, 0};
  if (live) {
    const int64_t step = static_cast<int64_t>(gy) * 8;
    int64_t r = static_cast<int64_t>(blockIdx.y) * 8 + ty;
    for (; r + 3 * step < rows; r += 4 * step) {
      uint4 h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) h[q] = Loader<DT>::template load8<true>(x, (r + q * step) * cols + cu * 8);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t w[4] = {h[q].x, h[q].y, h[q].z, h[q].w};
        if (SUM) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            acc[j] = __dadd_rn(acc[j], absh_to_f64((w[j >> 1] >> ((j & 1) * 16)) & 0xffffu));
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
        for (int j = 0; j < 8; ++j)
          acc[j] = __dadd_rn(acc[j], absh_to_f64((w[j >> 1] >> ((j & 1) * 16)) & 0xffffu));
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) mx[j] = __vmaxu2(mx[j], w[j] & 0x7fff7fffu);
      }
    }
  }
  if (SUM) {
#pragma unroll
    for (int j = 0; j < 8; ++j) red[ty][tx][j] = acc[j];
  } else {
    uint32_t *redu = reinterpret_cast<uint32_t *>(&red[0][0][0]);
#pragma unroll
    for (int j = 0; j < 4; ++j) redu[(ty * 32 + tx) * 4 + j] = mx[j];
  }
  __syncthreads();
  if (ty == 0 && live) {
    if (SUM) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = red[0][tx][j];
#pragma unroll
        for (int t = 1; t < 8; ++t) v[j] = __dadd_rn(v[j], red[t][tx][j]);
      }
      double *dst = a.partial + static_cast<int64_t>(blockIdx.y) * cols + cu * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) __stcg(dst + j, v[j]);
    } else {
      const uint32_t *redu = reinterpret_cast<const uint32_t *>(&red[0][0][0]);
      uint32_t *dst = reinterpret_cast<uint32_t *>(a.partial) + static_cast<int64_t>(blockIdx.y) * cols + cu * 8;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t v = redu[tx * 4 + j];
#pragma unroll
        for (int t = 1; t < 8; ++t) v = __vmaxu2(v, redu[(t * 32 + tx) * 4 + j]);
        __stcg(dst + 2 * j, v & 0xffffu);
        __stcg(dst + 2 * j + 1, v >> 16);
      }
    }
  }
  // ---- stage B: the last CTA of this column strip reduces the strip
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.strip_cnt + blockIdx.x, 1u) == static_cast<uint32_t>(gy - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kStripCols + threadIdx.x;
  if (c < cols) {
    if (SUM) {
      double s = 0.0;
      for (int b = 0; b < gy; ++b) s = __dadd_rn(s, __ldcg(a.partial + static_cast<int64_t>(b) * cols + c));
      __stcg(a.S + c, s);
      if (!(s < kExactLimit)) atomicOr(a.done_cnt + 1, 1u);
    } else {
      const uint32_t *p = reinterpret_cast<const uint32_t *>(a.partial);
      uint32_t m = 0;
      for (int b = 0; b < gy; ++b) m = max(m, __ldcg(p + static_cast<int64_t>(b) * cols + c));
      __stcg(a.colmax + c, m);
      if (m >= 0x7c00u && a.err) atomicOr(a.err, ADC_ERR_NONFINITE);
    }
  }
  if (threadIdx.x == 0) a.strip_cnt[blockIdx.x] = 0;  // reset for the next call
  if (!SUM) return;
  // ---- stage C: the last strip computes the statistics
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.done_cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) a.done_cnt[0] = 0;
  if (*(volatile uint32_t *)(a.done_cnt + 1)) {
    // numpy's row-order float64 sums (only when some total >= 2^29)
    for (int64_t cc = threadIdx.x; cc < cols; cc += blockDim.x) {
      double s = 0.0;
      for (int64_t r = 0; r < rows; ++r)
        s = __dadd_rn(s, fabs(static_cast<double>(h2f(Loader<DT>::load1(x, r * cols + cc)))));
      __stcg(a.S + cc, s);
    }
    __syncthreads();
    if (threadIdx.x == 0) a.done_cnt[1] = 0;
  }
  __syncthreads();
  if (a.do_stats)
    outlier_stats_block(a.S, rows, cols, a.thr, a.k_cap, a.tree, a.flag, a.rank, a.idx, a.k_out,
                        a.err, a.too_many_check != 0);
}

// ---------------------------------------------------------------------------
// generic path for unaligned / cols % 8 != 0 matrices: one thread per column
// accumulates in row order (always numpy-exact), then the same stats block.
// ---------------------------------------------------------------------------
template <int DT, bool SUM>
__global__ void __launch_bounds__(kThreads) colstats_generic(const void *__restrict__ x, ColArgs a) {
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
    outlier_stats_block(a.S, a.rows, a.cols, a.thr, a.k_cap, a.tree, a.flag, a.rank, a.idx,
                        a.k_out, a.err, a.too_many_check != 0);
}

// ---------------------------------------------------------------------------
#define ADC_DT_SWITCH(dt, DT, ...)                                   \
  switch (dt) {                                                      \
    case ADC_F32: { constexpr int DT = ADC_F32; __VA_ARGS__; break; }  \
    case ADC_BF16: { constexpr int DT = ADC_BF16; __VA_ARGS__; break; } \
    case ADC_F16: { constexpr int DT = ADC_F16; __VA_ARGS__; break; }  \
    default: return -1;                                              \
  }

static ColArgs make_args(int64_t rows, int64_t cols, const Workspace &ws) {
  ColArgs a{};
  a.rows = rows;
  a.cols = cols;
  a.partial = ws.partial;
  a.S = ws.colsum;
  a.colmax = ws.colmax;
  a.strip_cnt = ws.counters;
  a.done_cnt = ws.counters + ws.n_strips;
  a.tree = Tree{ws.node_lo, ws.node_n, ws.node_left, ws.node_val};
  a.flag = ws.flag;
  a.rank = ws.rank;
  return a;
}

static bool fast_cols(const void *x, int64_t cols) {
  return cols % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
}

static dim3 col_grid(const Ctx &c, int64_t rows, int64_t cols) {
  dim3 g(static_cast<unsigned>((cols + kStripCols - 1) / kStripCols), 1);
  int64_t want = (static_cast<int64_t>(c.num_sms) * 4 + g.x - 1) / g.x;
  const int64_t maxy = (rows + 7) / 8;
  if (want > kMaxRowBlocks) want = kMaxRowBlocks;
  if (want > maxy) want = maxy;
  g.y = static_cast<unsigned>(want < 1 ? 1 : want);
  return g;
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
    const dim3 g = col_grid(c, rows, cols);
    ADC_DT_SWITCH(dt, DT, (colstats<DT, true><<<g, kThreads, 0, c.stream>>>(x, a), note_launches(1)));
  } else {
    const int g = static_cast<int>((cols + kThreads - 1) / kThreads);
    ADC_DT_SWITCH(dt, DT, (colstats_generic<DT, true><<<g, kThreads, 0, c.stream>>>(x, a), note_launches(1)));
  }
  return 0;
}

int launch_colstats_max(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                        const Workspace &ws, uint32_t *err) {
  ColArgs a = make_args(rows, cols, ws);
  a.err = err;
  if (fast_cols(x, cols)) {
    const dim3 g = col_grid(c, rows, cols);
    ADC_DT_SWITCH(dt, DT, (colstats<DT, false><<<g, kThreads, 0, c.stream>>>(x, a), note_launches(1)));
  } else {
    const int g = static_cast<int>((cols + kThreads - 1) / kThreads);
    ADC_DT_SWITCH(dt, DT, (colstats_generic<DT, false><<<g, kThreads, 0, c.stream>>>(x, a), note_launches(1)));
  }
  return 0;
}

}  // namespace adc
