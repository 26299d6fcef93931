// K4 detection half: exact channel |x|-sums and the numpy-identical z-score.
//
// Reference: channel_abs_sums (codec.py:289-291), detect_outlier_channels
// (:294-305), the TooManyOutliers guard and index layout of
// compress_outlier_separated (:321-341).
//
// Exactness argument: every f16 value is an integer
// multiple of 2^-24 below 2^16, so float64 partial sums are exact -- and hence
// independent of summation order -- while the column total is < 2^29.  The
// parallel kernel therefore accumulates in any order (per-thread DADD, then
// atomicAdd(double)); a column whose running total reaches 2^29 raises a flag
// and `colsum_sequential` recomputes every column in numpy's row order.
// The mean / std / z-score use numpy's pairwise summation tree (block 128,
// unroll 8, initial 0.0), restated in oracle/codec_oracle.py:pairwise_sum and
// pinned there against ndarray.sum; all float64 ops use explicit _rn
// intrinsics so nothing is contracted into an FMA.
#include "common.cuh"
#include "launch.h"

namespace adc {

constexpr double kExactLimit = 536870912.0;  // 2^29

// |f16| -> f64 without the conversion pipe: f16 -> f32 (HADD2.F32), then
// re-bias the f32 exponent into an f64 (every f16 value is a normal f32).
__device__ __forceinline__ double absh_to_f64(uint32_t bits) {
  const uint32_t u = __float_as_uint(h2f(bits & 0x7fffu));
  const uint32_t hi = u ? (u >> 3) + (896u << 20) : 0u;
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
}

template <int DT>
__global__ void __launch_bounds__(kThreads)
    colsum_parallel(const void *__restrict__ x, int64_t rows, int64_t cols,
                    double *__restrict__ colsum, uint32_t *__restrict__ misc) {
  __shared__ double red[8][32][8];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t cu = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  const bool live = cu * 8 < cols;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (live) {
    for (int64_t r = static_cast<int64_t>(blockIdx.y) * 8 + ty; r < rows;
         r += static_cast<int64_t>(gridDim.y) * 8) {
      const uint4 h = Loader<DT>::template load8<true>(x, r * cols + cu * 8);
      const uint32_t w[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
      for (int j = 0; j < 8; ++j)
        acc[j] = __dadd_rn(acc[j], absh_to_f64((w[j >> 1] >> ((j & 1) * 16)) & 0xffffu));
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[ty][tx][j] = acc[j];
  __syncthreads();
  if (ty == 0 && live) {
    bool big = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double v = red[0][tx][j];
#pragma unroll
      for (int t = 1; t < 8; ++t) v = __dadd_rn(v, red[t][tx][j]);
      if (v != 0.0) {
        const double old = atomicAdd(colsum + cu * 8 + j, v);
        big |= !(__dadd_rn(old, v) < kExactLimit);
      }
    }
    if (big) atomicOr(misc, 1u);
  }
}

// numpy's row-order float64 sum, used only when some column total >= 2^29.
template <int DT>
__global__ void __launch_bounds__(kThreads)
    colsum_sequential(const void *__restrict__ x, int64_t rows, int64_t cols,
                      double *__restrict__ colsum, const uint32_t *__restrict__ misc) {
  if (*(volatile const uint32_t *)misc == 0) return;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; c < cols;
       c += static_cast<int64_t>(gridDim.x) * kThreads) {
    double acc = 0.0;
    for (int64_t r = 0; r < rows; ++r)
      acc = __dadd_rn(acc, fabs(static_cast<double>(h2f(Loader<DT>::load1(x, r * cols + c)))));
    colsum[c] = acc;
  }
}

// ---------------------------------------------------------------------------
// numpy pairwise summation (pairwise_sum_DOUBLE), split into parallel leaves
// ---------------------------------------------------------------------------
constexpr int64_t kBlock = 128;

struct Term {  // value of element i fed to the sum: S[i] or (S[i]-mean)^2
  const double *s;
  double mean;
  bool squared;
  __device__ __forceinline__ double operator()(int64_t i) const {
    if (!squared) return s[i];
    const double d = __dsub_rn(s[i], mean);
    return __dmul_rn(d, d);
  }
};

__device__ double leaf_sum(const Term &t, int64_t lo, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, t(lo + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = t(lo + j);
  int64_t i = 8;
  const int64_t stop = n - (n % 8);
  for (; i < stop; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], t(lo + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, t(lo + i));
  return res;
}

// The recursion of pairwise_sum_DOUBLE is evaluated without device recursion
// (no dynamic stack): thread 0 walks the tree with explicit shared-memory
// stacks, first to list the leaves left to right, later to add the leaf sums
// back up in exactly the recursion's order.
constexpr int kStackCap = 160;  // >= 2*depth+2; depth <= log2(n/57) < 64 for any int64 n

__device__ int64_t enumerate_leaves(int64_t n, int64_t *leaf, int64_t *st_lo, int64_t *st_n) {
  int sp = 0;
  int64_t count = 0;
  st_lo[sp] = 0;
  st_n[sp++] = n;
  while (sp) {
    --sp;
    const int64_t lo = st_lo[sp], m = st_n[sp];
    if (m <= kBlock) {
      leaf[count++] = (lo << 8) | m;
      continue;
    }
    int64_t h = m / 2;
    h -= h % 8;
    st_lo[sp] = lo + h;  // right pushed first: the left subtree is visited first
    st_n[sp++] = m - h;
    st_lo[sp] = lo;
    st_n[sp++] = h;
  }
  return count;
}

// Post-order evaluation: node entries are n (to expand) or -1 (combine marker).
__device__ double combine_tree(int64_t n, const double *leafsum, int64_t *st_n, double *vals) {
  int sp = 0, vp = 0;
  int64_t li = 0;
  st_n[sp++] = n;
  while (sp) {
    const int64_t m = st_n[--sp];
    if (m < 0) {
      const double b = vals[--vp];
      const double a = vals[--vp];
      vals[vp++] = __dadd_rn(a, b);
      continue;
    }
    if (m <= kBlock) {
      vals[vp++] = leafsum[li++];
      continue;
    }
    int64_t h = m / 2;
    h -= h % 8;
    st_n[sp++] = -1;
    st_n[sp++] = m - h;
    st_n[sp++] = h;
  }
  return vals[0];
}

constexpr int kStatsThreads = 1024;

__global__ void __launch_bounds__(kStatsThreads)
    outlier_stats(int64_t rows, int64_t cols, double thr, int64_t k_cap, const double *__restrict__ S,
                  int64_t *__restrict__ leaf, double *__restrict__ leafsum,
                  uint8_t *__restrict__ flag, int32_t *__restrict__ rank, uint32_t *__restrict__ idx,
                  int32_t *__restrict__ k_out, uint32_t *__restrict__ err, int too_many_check) {
  __shared__ int64_t s_nleaves;
  __shared__ double s_mean, s_sigma;
  __shared__ int s_bad;
  __shared__ int64_t s_warp[kStatsThreads / 32];
  __shared__ int64_t st_a[kStackCap], st_b[kStackCap];
  __shared__ double st_v[kStackCap];
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_nleaves = enumerate_leaves(cols, leaf, st_a, st_b);
    s_bad = 0;
  }
  __syncthreads();
  const int64_t nl = s_nleaves;
  // non-finite input shows up as a column sum no finite f16 matrix can reach
  const double cap = 65504.0 * static_cast<double>(rows);
  for (int64_t c = tid; c < cols; c += kStatsThreads)
    if (!(S[c] <= cap)) s_bad = 1;
  Term t{S, 0.0, false};
  for (int64_t l = tid; l < nl; l += kStatsThreads)
    leafsum[l] = leaf_sum(t, leaf[l] >> 8, leaf[l] & 0xff);
  __syncthreads();
  if (tid == 0) {
    const double tot = __dadd_rn(0.0, combine_tree(cols, leafsum, st_a, st_v));
    s_mean = __ddiv_rn(tot, static_cast<double>(cols));
  }
  __syncthreads();
  t.mean = s_mean;
  t.squared = true;
  for (int64_t l = tid; l < nl; l += kStatsThreads)
    leafsum[l] = leaf_sum(t, leaf[l] >> 8, leaf[l] & 0xff);
  __syncthreads();
  if (tid == 0) {
    const double tot = __dadd_rn(0.0, combine_tree(cols, leafsum, st_a, st_v));
    s_sigma = __dsqrt_rn(__ddiv_rn(tot, static_cast<double>(cols)));
    if (s_bad && err) atomicOr(err, ADC_ERR_NONFINITE);
  }
  __syncthreads();
  const double mean = s_mean, sigma = s_sigma;
  // flags + stable compaction: each thread owns a contiguous run of columns
  const int64_t chunk = (cols + kStatsThreads - 1) / kStatsThreads;
  const int64_t c_lo = min(cols, chunk * tid), c_hi = min(cols, c_lo + chunk);
  int64_t mine = 0;
  for (int64_t c = c_lo; c < c_hi; ++c) {
    const bool f = sigma != 0.0 && __ddiv_rn(__dsub_rn(S[c], mean), sigma) > thr;
    flag[c] = f;
    mine += f;
  }
  // block exclusive scan of `mine`
  const int lane = tid & 31, wid = tid >> 5;
  int64_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int64_t v = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    s_warp[lane] = v;  // inclusive over warps
  }
  __syncthreads();
  int64_t pos = incl - mine + (wid ? s_warp[wid - 1] : 0);
  for (int64_t c = c_lo; c < c_hi; ++c) {
    if (flag[c]) {
      rank[c] = static_cast<int32_t>(pos);
      if (pos < k_cap) idx[pos] = static_cast<uint32_t>(c);
      ++pos;
    } else {
      rank[c] = -1;
    }
  }
  if (tid == kStatsThreads - 1) {
    const int64_t k = s_warp[31];
    *k_out = static_cast<int32_t>(k);
    if (err) {
      if (too_many_check && 2 * k > cols) atomicOr(err, ADC_ERR_TOO_MANY_OUTLIERS);
      if (k > k_cap) atomicOr(err, ADC_ERR_K_CAP);
    }
  }
}

__global__ void copy_sums(const double *__restrict__ s, double *__restrict__ out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = s[i];
}

// ---------------------------------------------------------------------------
#define ADC_DT_SWITCH(dt, DT, ...)                                   \
  switch (dt) {                                                      \
    case ADC_F32: { constexpr int DT = ADC_F32; __VA_ARGS__; break; }  \
    case ADC_BF16: { constexpr int DT = ADC_BF16; __VA_ARGS__; break; } \
    case ADC_F16: { constexpr int DT = ADC_F16; __VA_ARGS__; break; }  \
    default: return -1;                                              \
  }

template <int DT>
__global__ void __launch_bounds__(kThreads)
    colsum_generic(const void *__restrict__ x, int64_t rows, int64_t cols,
                   double *__restrict__ colsum, uint32_t *__restrict__ misc) {
  // one thread per column, any alignment; exactness flag as in the fast path
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; c < cols;
       c += static_cast<int64_t>(gridDim.x) * kThreads) {
    double acc = 0.0;
    for (int64_t r = 0; r < rows; ++r)
      acc = __dadd_rn(acc, absh_to_f64(Loader<DT>::load1(x, r * cols + c)));
    colsum[c] = acc;
    if (!(acc < kExactLimit)) atomicOr(misc, 1u);
  }
}

int launch_colsum(const Ctx &c, const void *x, int dt, int64_t rows, int64_t cols,
                  const Workspace &ws, uint32_t *err) {
  (void)err;
  if (cudaMemsetAsync(ws.colsum, 0, sizeof(double) * cols, c.stream) != cudaSuccess) return -2;
  if (cudaMemsetAsync(ws.misc, 0, sizeof(uint32_t) * 4, c.stream) != cudaSuccess) return -2;
  const bool fast = cols % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
  const int gs = static_cast<int>((cols + kThreads - 1) / kThreads);
  if (fast) {
    dim3 g(static_cast<unsigned>((cols / 8 + 31) / 32), 1);
    int64_t want = static_cast<int64_t>(c.num_sms) * 8 / g.x;
    int64_t maxy = (rows + 7) / 8;
    g.y = static_cast<unsigned>(want < 1 ? 1 : (want > maxy ? maxy : want));
    ADC_DT_SWITCH(dt, DT, {
      colsum_parallel<DT><<<g, kThreads, 0, c.stream>>>(x, rows, cols, ws.colsum, ws.misc), note_launches(1);
      colsum_sequential<DT><<<gs, kThreads, 0, c.stream>>>(x, rows, cols, ws.colsum, ws.misc), note_launches(1);
    });
  } else {
    ADC_DT_SWITCH(dt, DT, {
      colsum_generic<DT><<<gs, kThreads, 0, c.stream>>>(x, rows, cols, ws.colsum, ws.misc), note_launches(1);
      colsum_sequential<DT><<<gs, kThreads, 0, c.stream>>>(x, rows, cols, ws.colsum, ws.misc), note_launches(1);
    });
  }
  return 0;
}

int launch_outlier_stats(const Ctx &c, int64_t rows, int64_t cols, double thr, int64_t k_cap,
                         const Workspace &ws, uint32_t *idx, int32_t *k_out, uint32_t *err,
                         bool too_many_check) {
  outlier_stats<<<1, kStatsThreads, 0, c.stream>>>(rows, cols, thr, k_cap, ws.colsum, ws.leaf,
                                                   ws.leafsum, ws.flag, ws.rank, idx, k_out, err,
                                                   too_many_check ? 1 : 0), note_launches(1);
  return 0;
}

int launch_copy_sums(const Ctx &c, const Workspace &ws, double *out, int64_t cols) {
  copy_sums<<<static_cast<int>((cols + 255) / 256), 256, 0, c.stream>>>(ws.colsum, out, cols), note_launches(1);
  return 0;
}

}  // namespace adc
