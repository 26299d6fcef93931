// Block-level statistics shared by the column-statistics kernel (outlier.cu)
// and the fused outlier-separated kernel (fused.cu): numpy's pairwise
// summation tree evaluated level-parallel, the z-score flags and the ranks.
// See outlier.cu for the exactness argument.
#pragma once

#include <algorithm>
#include <functional>
#include <utility>
#include <vector>

#include "common.cuh"

namespace adc {

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

// tuning timestamps of the statistics phases (null: off)
__device__ __forceinline__ void stats_mark(unsigned long long *tm, int i, double dep = 0.0) {
  if (tm && threadIdx.x == 0) {
    unsigned long long t;
    // `dep` is an input operand: the value it names is computed before the
    // timestamp (pure arithmetic is otherwise free to move across it)
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "d"(dep));
    tm[i] = t;
  }
}

template <bool SMEM>
struct Term {  // element i of the summed vector: S[i] or (S[i]-mean)^2
  const double *s;  // shared memory (SMEM) or global memory written by this CTA
  double mean;
  bool squared;
  __device__ __forceinline__ double load(int64_t i) const { return SMEM ? s[i] : __ldcg(s + i); }
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
template <class T>
__device__ __forceinline__ double leaf_sum8(const T &t, int lo, int n, bool valid) {
  const int j = threadIdx.x & 7;
  const int stop = n - (n % 8);
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (valid && 8 * i + j < stop) ? t.load(lo + 8 * i + j) : 0.0;
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
    for (int i = stop; i < n; ++i) c = __dadd_rn(c, t.map(t.load(lo + i)));
  }
  return c;
}

// numpy's pairwise recursion splits n > 128 into h = n/2 - (n/2) % 8 and n - h.
__device__ __forceinline__ int pw_half(int n) {
  const int h = n / 2;
  return h - h % 8;
}

// ---- small vectors (n <= kHeapMaxCols): the tree in heap order, no build step.
// The right child is never smaller than the left, so the rightmost path is
// the deepest; for n <= 16384 leaves sit at depth <= 8 (511 heap slots).
constexpr int kHeapMaxCols = 16384;
constexpr int kHeapNodes = 511;

__device__ __forceinline__ int heap_depth(int n) {
  int d = 0;
  while (n > 128) {
    n -= pw_half(n);
    ++d;
  }
  return d;
}

// Walk from the root along the left/right choices in `path` (MSB first, d
// steps); returns false if a leaf is reached before depth d.
__device__ __forceinline__ bool heap_walk(int n, int path, int d, int &lo, int &m) {
  lo = 0;
  m = n;
  for (int l = d - 1; l >= 0; --l) {
    if (m <= 128) return false;
    const int h = pw_half(m);
    if ((path >> l) & 1) {
      lo += h;
      m -= h;
    } else {
      m = h;
    }
  }
  return true;
}

// pairwise_sum over the n terms of t; every thread of the block calls and
// receives the result.  Leaf slot g (of 2^D) follows the bits of g from the
// root; the first slot under each leaf evaluates it with 8 lanes.
template <class T>
__device__ __forceinline__ double heap_sum(const T &t, int n, int D, double *val) {
  const int slots = 1 << D;
  const int groups = blockDim.x / 8;
  for (int base = 0; base < slots; base += groups) {  // uniform trip count
    const int g = base + static_cast<int>(threadIdx.x) / 8;
    int lo = 0, m = 0, leaf = 0;
    bool own = false;
    if (g < slots) {
      // descend until a leaf; own it if the remaining path bits are zero
      m = n;
      int d = 0;
      while (m > 128) {
        const int hf = pw_half(m);
        if ((g >> (D - 1 - d)) & 1) {
          lo += hf;
          m -= hf;
          leaf = 2 * leaf + 2;
        } else {
          m = hf;
          leaf = 2 * leaf + 1;
        }
        ++d;
      }
      own = (g & ((1 << (D - d)) - 1)) == 0;
    }
    const double v = leaf_sum8(t, own ? lo : 0, own ? m : 0, own);
    if (own && (threadIdx.x & 7) == 0) val[leaf] = v;
  }
  __syncthreads();
  for (int d = D - 1; d >= 0; --d) {  // bottom-up over internal nodes
    const int i = static_cast<int>(threadIdx.x);
    if (i < (1 << d)) {
      int lo, m;
      if (heap_walk(n, i, d, lo, m) && m > 128) {
        const int hi = (1 << d) - 1 + i;
        val[hi] = __dadd_rn(val[2 * hi + 1], val[2 * hi + 2]);
      }
    }
    __syncthreads();
  }
  const double r = __dadd_rn(0.0, val[0]);
  __syncthreads();
  return r;
}

// ---- large vectors: level-parallel tree with the node arrays in the workspace.
struct Tree {
  int32_t *lo, *n, *left;
  double *val;
};

static __device__ int build_tree(int n, const Tree &tr, int *s_lvl, int *s_tmp) {
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
          const int h = pw_half(m);
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

template <class T>
static __device__ double tree_sum(const T &t, const Tree &tr, int depth, const int *s_lvl) {
  const int total_nodes = s_lvl[depth];
  const int groups = blockDim.x / 8;
  const int g = threadIdx.x / 8;
  for (int base = 0; base < total_nodes; base += groups) {
    const int i = base + g;
    const bool valid = i < total_nodes && __ldcg(tr.left + i) < 0;
    const double v = leaf_sum8(t, valid ? __ldcg(tr.lo + i) : 0, valid ? __ldcg(tr.n + i) : 0, valid);
    if (valid && (threadIdx.x & 7) == 0) tr.val[i] = v;
  }
  __threadfence_block();
  __syncthreads();
  for (int d = depth - 2; d >= 0; --d) {
    for (int i = s_lvl[d] + threadIdx.x; i < s_lvl[d + 1]; i += blockDim.x) {
      const int l = __ldcg(tr.left + i);
      if (l >= 0) __stcg(tr.val + i, __dadd_rn(__ldcg(tr.val + l), __ldcg(tr.val + l + 1)));
    }
    __threadfence_block();
    __syncthreads();
  }
  const double r = __dadd_rn(0.0, __ldcg(tr.val));
  __syncthreads();
  return r;
}

// The z-score flags, ranks and outputs of detect_outlier_channels /
// compress_outlier_separated given mean and population variance of S
// (codec.py:302-305, 321-341); all threads of the block call.
template <bool SMEM>
__device__ __forceinline__ int outlier_flags_block(Term<SMEM> t, double mean, double var,
                                                   int64_t rows, int64_t cols, double thr,
                                                   int64_t k_cap, uint8_t *flag, uint32_t *idx,
                                                   int32_t *k_out, uint32_t *err,
                                                   bool too_many_check, unsigned long long *tm = nullptr) {
  __shared__ int s_tmp[32];
  t.mean = mean;
  t.squared = false;
  const double sigma = __dsqrt_rn(var);
  const double cap = 65504.0 * static_cast<double>(rows);
  // z-score flag (strict >, codec.py:305); a sum above rows * 65504 means an
  // inf/NaN input (no finite f16 matrix reaches it).
  // q = fl(d / sigma) with d = fl(S - mean) is monotone in d (sigma > 0), so
  // q > thr is decided in the d domain against T = fl(thr * sigma): d beyond
  // T by more than |T| * 2^-46 (+ 2^-1000) puts the exact quotient beyond
  // thr by far more than q's half-ulp rounding, either way; only d inside
  // that margin (or NaN) pays for the correctly rounded division.  One DSUB
  // and two compares per column -- no reciprocal, no dependent chain.
  const double T = __dmul_rn(thr, sigma);
  const double T_m = __dadd_rn(__dmul_rn(fabs(T), 0x1p-46), 0x1p-1000);
  const double T_hi = __dadd_rn(T, T_m), T_lo = __dsub_rn(T, T_m);
  auto z_exact = [&](double v) -> uint32_t {
    return (sigma != 0.0 && __ddiv_rn(__dsub_rn(v, mean), sigma) > thr) ? 1u : 0u;
  };
  const int64_t run = (cols + blockDim.x - 1) / blockDim.x;
  const int64_t c0 = min(cols, run * threadIdx.x), c1 = min(cols, c0 + run);
  int bad = 0, mine = 0, total, pos;
  if (run <= 64) {
    // each thread owns a contiguous run of <= 64 columns: flags in a register
    // mask.  32-bit column indices (cols < 2^31 here), and the rare
    // ambiguous column re-reads its sum instead of indexing the batch array
    // at run time (which put the batch in local memory: 8 STL per batch)
    uint64_t bits = 0;
    const int i0 = static_cast<int>(c0), i1 = static_cast<int>(c1);
    for (int base = i0; base < i1; base += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = base + q < i1 ? t.load(base + q) : 0.0;
      uint32_t f8 = 0, amb = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double d = __dsub_rn(v[q], mean);
        const bool hi = d > T_hi, lo = d < T_lo;
        const bool live = base + q < i1;
        bad |= live && !(v[q] <= cap);
        f8 |= (live && hi && sigma != 0.0 ? 1u : 0u) << q;
        amb |= (live && !hi && !lo && sigma != 0.0 ? 1u : 0u) << q;
      }
      while (amb) {  // rare: within 2^-46 of the threshold (or NaN)
        const int q = __ffs(amb) - 1;
        amb &= amb - 1;
        f8 |= z_exact(t.load(base + q)) << q;
      }
      bits |= static_cast<uint64_t>(f8) << (base - i0);
    }
    stats_mark(tm, 2);
    bad = __syncthreads_or(bad);
    mine = __popcll(bits);
    pos = block_excl_scan(mine, &total, s_tmp);
    stats_mark(tm, 3);
    // graceful k_cap overflow: ranks >= k_cap stay in their groups
    uint64_t kept = bits;
    for (uint64_t m = bits; m; m &= m - 1, ++pos) {
      const int j = __ffsll(static_cast<long long>(m)) - 1;
      if (pos < k_cap) {
        if (idx) idx[pos] = static_cast<uint32_t>(c0 + j);
      } else {
        kept &= ~(1ull << j);
      }
    }
    if ((c0 & 3) == 0 && ((c1 - c0) & 3) == 0) {  // 4 flag bytes per store
      for (int64_t c = c0; c < c1; c += 4) {
        const uint32_t nib = static_cast<uint32_t>(kept >> (c - c0)) & 0xfu;
        const uint32_t word = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
        *reinterpret_cast<uint32_t *>(flag + c) = word;
      }
    } else {
      for (int64_t c = c0; c < c1; ++c) flag[c] = static_cast<uint8_t>((kept >> (c - c0)) & 1u);
    }
  } else {
    // very wide rows: flags through global memory
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const double v = t.load(c);
      bad |= !(v <= cap);
      flag[c] = static_cast<uint8_t>(z_exact(v));
    }
    bad = __syncthreads_or(bad);
    for (int64_t c = c0; c < c1; ++c) mine += flag[c];
    pos = block_excl_scan(mine, &total, s_tmp);
    for (int64_t c = c0; c < c1; ++c) {
      if (flag[c]) {
        if (pos < k_cap) {
          if (idx) idx[pos] = static_cast<uint32_t>(c);
        } else {
          flag[c] = 0;
        }
        ++pos;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (k_out) *k_out = total;
    if (err) {
      if (bad) atomicOr(err, ADC_ERR_NONFINITE);
      if (too_many_check && 2 * static_cast<int64_t>(total) > cols) atomicOr(err, ADC_ERR_TOO_MANY_OUTLIERS);
      if (total > k_cap) atomicOr(err, ADC_ERR_K_CAP);
    }
  }
  return total;
}

// Stage C: mean / std / z-score flags / indices (codec.py:294-305, 324-341).
// S is in shared memory (s_in_smem) or in global memory written by this CTA;
// `scratch` is >= kStatsScratch bytes of shared memory.  Outputs: flag[c]
// (0/1 bytes, global), the ascending indices idx[0 .. min(k, k_cap)), k and
// the error bits.  Columns ranked >= k_cap stay in their groups (flag 0):
// graceful overflow, reported by ADC_ERR_K_CAP.  Returns k to every thread.
constexpr int kStatsScratch = kHeapNodes * 8 + 8;
template <bool SMEM>
__device__ __forceinline__ int outlier_stats_block(const double *S, int64_t rows,
                                           int64_t cols, double thr, int64_t k_cap,
                                           const Tree &tr, uint8_t *flag, uint32_t *idx,
                                           int32_t *k_out, uint32_t *err, bool too_many_check,
                                           unsigned char *scratch, unsigned long long *tm = nullptr) {
  __shared__ int s_lvl[72];
  __shared__ int s_tmp[32];
  const int n = static_cast<int>(cols);
  Term<SMEM> t{S, 0.0, false};
  double mean, var;
  if (cols <= kHeapMaxCols) {
    double *val = reinterpret_cast<double *>(scratch);
    const int D = heap_depth(n);
    // the mean's sum: when the any-order total stays below 2^29 every partial
    // sum of numpy's tree is exact (non-negative multiples of 2^-24), so the
    // tree equals a plain block reduction (see warp_mean_var)
    double part = 0.0;
    // 8 loads in flight per thread (S may be in global memory: one L2 round
    // trip per batch instead of per column; the sum is exact in any order)
    for (int64_t c0 = threadIdx.x; c0 < cols; c0 += 8 * static_cast<int64_t>(blockDim.x)) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t c = c0 + q * static_cast<int64_t>(blockDim.x);
        v[q] = c < cols ? t.load(c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) part = __dadd_rn(part, v[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
    if ((threadIdx.x & 31) == 0) val[threadIdx.x >> 5] = part;
    __syncthreads();
    // the warp partials combined as a tree (exact, so any order)
    double wv[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) wv[w] = w < static_cast<int>(blockDim.x >> 5) ? val[w] : 0.0;
    double total = __dadd_rn(__dadd_rn(__dadd_rn(wv[0], wv[1]), __dadd_rn(wv[2], wv[3])),
                             __dadd_rn(__dadd_rn(wv[4], wv[5]), __dadd_rn(wv[6], wv[7])));
    for (int w = 8; w < static_cast<int>(blockDim.x >> 5); ++w) total = __dadd_rn(total, val[w]);
    __syncthreads();
    if (!(total < 536870912.0)) total = heap_sum(t, n, D, val);
    mean = __ddiv_rn(__dadd_rn(0.0, total), static_cast<double>(cols));
    stats_mark(tm, 0, mean);
    t.mean = mean;
    t.squared = true;
    var = __ddiv_rn(heap_sum(t, n, D, val), static_cast<double>(cols));
    stats_mark(tm, 1, var);
  } else {
    const int depth = build_tree(n, tr, s_lvl, s_tmp);
    mean = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
    t.mean = mean;
    t.squared = true;
    var = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
  }
  return outlier_flags_block(t, mean, var, rows, cols, thr, k_cap, flag, idx, k_out, err,
                             too_many_check, tm);
}

}  // namespace adc
