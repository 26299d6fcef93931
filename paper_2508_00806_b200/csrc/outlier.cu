// K4 detection half: exact channel |x|-sums and the numpy-identical z-score,
// plus the per-channel abs-max pass of K3 -- one kernel launch each.
//
// Reference: channel_abs_sums (codec.py:289-291), detect_outlier_channels
// (:294-305), the TooManyOutliers guard and index layout of
// compress_outlier_separated (:321-341); per-channel scales (:181-182, 225-227).
//
// One launch, three stages, chained with the last-block-done pattern (no grid
// barrier, no cooperative launch, no global atomics on data):
//   A. every CTA reduces a (rows/gy) x 256-column tile into column partials;
//      the 8 CTAs of a thread-block cluster (stacked along rows) combine
//      theirs through distributed shared memory and write one partial;
//   B. the last cluster to finish in a column strip sums that strip's partials;
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
#include <cooperative_groups.h>

#include "common.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace adc {

constexpr int kClusterY = 8;  // CTAs per cluster, stacked along rows

constexpr double kExactLimit = 536870912.0;  // 2^29
constexpr int kStripCols = 256;              // 32 column units of 8 per CTA

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
  __device__ __forceinline__ double map(double v) const {
    if (!squared) return v;
    const double d = __dsub_rn(v, mean);
    return __dmul_rn(d, d);
  }
};

// One leaf (n <= 128) of pairwise_sum_DOUBLE computed by an aligned group of
// 8 lanes: lane j owns accumulator r[j] = a[j] + a[j+8] + ... (in order); the
// final ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) is built with width-8 shuffles in
// exactly that order; lane 0 adds the n % 8 remainder sequentially.  The 16
// loads of a lane are issued together (one L2 round trip).  All 32 lanes call.
__device__ __forceinline__ double leaf_sum8(const Term &t, int lo, int n, bool valid) {
  const int j = threadIdx.x & 7;
  const int stop = n - (n % 8);
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (valid && 8 * i + j < stop) ? __ldcg(t.s + lo + 8 * i + j) : 0.0;
  double res = 0.0;
  if (valid && n >= 8) {
    double r = t.map(v[0]);
#pragma unroll
    for (int i = 1; i < 16; ++i)
      if (8 * i < stop) r = __dadd_rn(r, t.map(v[i]));
    res = r;
  }
  const double a = __dadd_rn(res, __shfl_down_sync(0xffffffffu, res, 1, 8));
  const double b = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, 2, 8));
  double c = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, 4, 8));
  if (valid && j == 0) {
    if (n < 8) c = 0.0;
    for (int i = stop; i < n; ++i) c = __dadd_rn(c, t.map(__ldcg(t.s + lo + i)));
  }
  return c;
}

// Level-parallel evaluation of numpy's pairwise recursion over n values.
// Node arrays live in shared memory when they fit, else in the workspace.
struct Tree {
  int32_t *lo, *n, *left;
  double *val;
};
constexpr int kSmemNodes = 1024;  // enough for n <= 16384 (leaves hold >= 56 values)

__device__ int build_tree(int n, const Tree &tr, int *s_lvl, int *s_tmp) {
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
      const int m = i < e ? tr.n[i] : 0;
      const int internal = (i < e && m > 128) ? 1 : 0;
      int total;
      const int before = block_excl_scan(internal, &total, s_tmp);
      if (i < e) {
        if (internal) {
          const int l = next + 2 * before;
          const int lo = tr.lo[i];
          int h = m / 2;
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
  const double r = __dadd_rn(0.0, tr.val[0]);
  __syncthreads();
  return r;
}

// Stage C: mean / std / z-score flags / ranks / indices (codec.py:294-305, 324-341).
// `scratch` is >= kStatsScratch bytes of shared memory (the stage-A buffers,
// no longer live): tree nodes + a flag byte per column when cols <= 16384.
constexpr int kStatsScratch = kSmemNodes * 20 + 16384;
__device__ void outlier_stats_block(const double *S, int64_t rows, int64_t cols, double thr,
                                    int64_t k_cap, const Tree &tr_global, uint8_t *flag,
                                    int32_t *rank, uint32_t *idx, int32_t *k_out, uint32_t *err,
                                    bool too_many_check, unsigned char *scratch) {
  __shared__ int s_lvl[72];
  __shared__ int s_tmp[32];
  const bool small = cols <= 16384;
  const Tree tr = small ? Tree{reinterpret_cast<int32_t *>(scratch),
                               reinterpret_cast<int32_t *>(scratch + 4 * kSmemNodes),
                               reinterpret_cast<int32_t *>(scratch + 8 * kSmemNodes),
                               reinterpret_cast<double *>(scratch + 12 * kSmemNodes)}
                        : tr_global;
  uint8_t *sflag = small ? scratch + 20 * kSmemNodes : flag;
  const int depth = build_tree(static_cast<int>(cols), tr, s_lvl, s_tmp);
  Term t{S, 0.0, false};
  const double mean = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
  t.mean = mean;
  t.squared = true;
  const double var = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
  const double sigma = __dsqrt_rn(var);
  // pass 1, coalesced and batched: z-score flags (strict >, codec.py:305)
  const double cap = 65504.0 * static_cast<double>(rows);
  int bad = 0;
  for (int64_t base = 0; base < cols; base += 8 * static_cast<int64_t>(blockDim.x)) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t c = base + q * blockDim.x + threadIdx.x;
      v[q] = c < cols ? __ldcg(S + c) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t c = base + q * blockDim.x + threadIdx.x;
      if (c < cols) {
        bad |= !(v[q] <= cap);  // inf/NaN input: no finite f16 matrix reaches this sum
        const bool f = sigma != 0.0 && __ddiv_rn(__dsub_rn(v[q], mean), sigma) > thr;
        sflag[c] = f ? 1 : 0;
        if (small) flag[c] = f ? 1 : 0;
      }
    }
  }
  bad = __syncthreads_or(bad);
  // pass 2: contiguous runs -> one block scan -> ranks and ascending indices
  const int64_t run = (cols + blockDim.x - 1) / blockDim.x;
  const int64_t c0 = min(cols, run * threadIdx.x), c1 = min(cols, c0 + run);
  int mine = 0;
  for (int64_t c = c0; c < c1; ++c) mine += sflag[c];
  int total;
  int pos = block_excl_scan(mine, &total, s_tmp);
  for (int64_t c = c0; c < c1; ++c) {
    if (sflag[c]) {
      rank[c] = pos;
      if (pos < k_cap)
        idx[pos] = static_cast<uint32_t>(c);
      else
        flag[c] = 0;  // beyond the side buffer: left in its groups (graceful overflow)
      ++pos;
    } else {
      rank[c] = -1;
    }
  }
  if (threadIdx.x == 0) {
    *k_out = total;
    if (err) {
      if (bad) atomicOr(err, ADC_ERR_NONFINITE);
      if (too_many_check && 2 * static_cast<int64_t>(total) > cols) atomicOr(err, ADC_ERR_TOO_MANY_OUTLIERS);
      if (total > k_cap) atomicOr(err, ADC_ERR_K_CAP);
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
__global__ void __cluster_dims__(1, kClusterY, 1) __launch_bounds__(kThreads, 3)
    colstats(const void *__restrict__ x, ColArgs a) {
  // stage A/B buffers and the stage-C scratch share one allocation
  __shared__ __align__(16) unsigned char s_raw[kStatsScratch > 18432 ? kStatsScratch : 18432];
  double(*red)[32][8] = reinterpret_cast<double(*)[32][8]>(s_raw);
  double *cpart = reinterpret_cast<double *>(s_raw + 16384);
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
  if (SUM) {
#pragma unroll
    for (int j = 0; j < 8; ++j) red[ty][tx][j] = acc[j];
  } else {
    uint32_t *redu = reinterpret_cast<uint32_t *>(&red[0][0][0]);
#pragma unroll
    for (int j = 0; j < 4; ++j) redu[(ty * 32 + tx) * 4 + j] = mx[j];
  }
  __syncthreads();
  // block partial of strip column t = 8*tx + j: reduce the 8 row lanes
  {
    const int t = threadIdx.x, ctx = t >> 3, cj = t & 7;
    if (SUM) {
      double v = red[0][ctx][cj];
#pragma unroll
      for (int q = 1; q < 8; ++q) v = __dadd_rn(v, red[q][ctx][cj]);
      cpart[t] = v;
    } else {
      const uint32_t *redu = reinterpret_cast<const uint32_t *>(&red[0][0][0]);
      uint32_t v = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) v = max(v, (redu[(q * 32 + ctx) * 4 + (cj >> 1)] >> (16 * (cj & 1))) & 0xffffu);
      reinterpret_cast<uint32_t *>(cpart)[t] = v;
    }
  }
  // cluster reduction over the kClusterY CTAs stacked along rows (DSMEM)
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kStripCols + threadIdx.x;
  const int64_t crow = blockIdx.y / kClusterY;
  if (cluster.block_rank() == 0 && c < cols) {
    if (SUM) {
      double v[kClusterY];
#pragma unroll
      for (int r = 0; r < kClusterY; ++r) v[r] = *cluster.map_shared_rank(cpart + threadIdx.x, r);
      double sum = v[0];
#pragma unroll
      for (int r = 1; r < kClusterY; ++r) sum = __dadd_rn(sum, v[r]);
      __stcg(a.partial + crow * cols + c, sum);
    } else {
      uint32_t *cpu = reinterpret_cast<uint32_t *>(cpart);
      uint32_t m = 0;
#pragma unroll
      for (int r = 0; r < kClusterY; ++r) m = max(m, *cluster.map_shared_rank(cpu + threadIdx.x, r));
      __stcg(reinterpret_cast<uint32_t *>(a.partial) + crow * cols + c, m);
    }
  }
  cluster.sync();  // peers' shared memory must outlive rank 0's reads
  if (cluster.block_rank() != 0) return;
  // ---- stage B: the last cluster of this column strip reduces the strip
  const int gyc = gy / kClusterY;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.strip_cnt + blockIdx.x, 1u) == static_cast<uint32_t>(gyc - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (c < cols) {
    if (SUM) {
      double p4[4] = {0.0, 0.0, 0.0, 0.0};
      int b = 0;
      for (; b + 4 <= gyc; b += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          p4[q] = __dadd_rn(p4[q], __ldcg(a.partial + static_cast<int64_t>(b + q) * cols + c));
      }
      for (; b < gyc; ++b) p4[0] = __dadd_rn(p4[0], __ldcg(a.partial + static_cast<int64_t>(b) * cols + c));
      const double s = __dadd_rn(__dadd_rn(p4[0], p4[1]), __dadd_rn(p4[2], p4[3]));
      __stcg(a.S + c, s);
      if (!(s < kExactLimit)) atomicOr(a.done_cnt + 1, 1u);
    } else {
      const uint32_t *p = reinterpret_cast<const uint32_t *>(a.partial);
      uint32_t m = 0;
      for (int b = 0; b < gyc; ++b) m = max(m, __ldcg(p + static_cast<int64_t>(b) * cols + c));
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
                        a.err, a.too_many_check != 0, s_raw);
}

// ---------------------------------------------------------------------------
// generic path for unaligned / cols % 8 != 0 matrices: one thread per column
// accumulates in row order (always numpy-exact), then the same stats block.
// ---------------------------------------------------------------------------
template <int DT, bool SUM>
__global__ void __launch_bounds__(kThreads) colstats_generic(const void *__restrict__ x, ColArgs a) {
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
    outlier_stats_block(a.S, a.rows, a.cols, a.thr, a.k_cap, a.tree, a.flag, a.rank, a.idx,
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
  // many short CTAs (measured: gy = 128 beats one wave of long CTAs: the
  // tail of a partial second wave costs more than the extra partials)
  (void)c;
  int64_t want = kMaxRowBlocks;
  const int64_t maxy = (rows + 7) / 8;
  if (want > kMaxRowBlocks) want = kMaxRowBlocks;
  if (want > maxy) want = maxy;
  want = (want + kClusterY - 1) / kClusterY * kClusterY;  // whole clusters
  g.y = static_cast<unsigned>(want < kClusterY ? kClusterY : want);
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
