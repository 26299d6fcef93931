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

// ---- one warp, host-built tree (fused.cu): numpy's pairwise recursion for a
// fixed length n <= 4096 flattened into leaves (left to right) and internal
// nodes sorted by height, so one warp evaluates it with no block barrier.
constexpr int kPwMaxLeaves = 40;
struct PwTree {
  int n_leaves, n_levels;
  int16_t leaf_lo[kPwMaxLeaves], leaf_n[kPwMaxLeaves];
  uint8_t left[kPwMaxLeaves], right[kPwMaxLeaves];  // internal node j = id n_leaves + j
  uint8_t level_end[8];                              // internal nodes of height <= h+1: [0, level_end[h])
};

// numpy's pairwise recursion (split n > 128 at n/2 - (n/2) % 8) flattened for
// warp_tree_sum: leaves left to right, internal nodes ordered by height.
inline bool build_pw_tree(int n, PwTree &t) {
  struct Internal { int l, r, h; };
  std::vector<Internal> in;
  std::vector<std::pair<int, int>> leaves;
  // returns (encoded id, height); leaves encoded >= 0, internal as -(k + 1)
  std::function<std::pair<int, int>(int, int)> rec = [&](int lo, int m) -> std::pair<int, int> {
    if (m <= 128) {
      leaves.emplace_back(lo, m);
      return {static_cast<int>(leaves.size()) - 1, 0};
    }
    const int h = m / 2 - (m / 2) % 8;
    const auto a = rec(lo, h), b = rec(lo + h, m - h);
    in.push_back({a.first, b.first, 1 + std::max(a.second, b.second)});
    return {-static_cast<int>(in.size()), in.back().h};
  };
  rec(0, n);
  const int nl = static_cast<int>(leaves.size()), ni = static_cast<int>(in.size());
  if (nl > kPwMaxLeaves || ni >= kPwMaxLeaves) return false;
  std::vector<int> order(ni), pos(ni);
  for (int i = 0; i < ni; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return in[x].h < in[y].h; });
  for (int i = 0; i < ni; ++i) pos[order[i]] = i;
  auto id = [&](int enc) { return enc >= 0 ? enc : nl + pos[-enc - 1]; };
  t = PwTree{};
  t.n_leaves = nl;
  for (int i = 0; i < nl; ++i) {
    t.leaf_lo[i] = static_cast<int16_t>(leaves[i].first);
    t.leaf_n[i] = static_cast<int16_t>(leaves[i].second);
  }
  int levels = 0;
  for (int j = 0; j < ni; ++j) {
    const Internal &v = in[order[j]];
    t.left[j] = static_cast<uint8_t>(id(v.l));
    t.right[j] = static_cast<uint8_t>(id(v.r));
    levels = std::max(levels, v.h);
    t.level_end[v.h - 1] = static_cast<uint8_t>(j + 1);
  }
  t.n_levels = levels;
  return levels <= 8;
}

// pairwise_sum of the terms of t by warp 0 (all 32 lanes call); val holds
// >= 2 * kPwMaxLeaves doubles of shared memory.  Returns 0.0 + sum (as the
// block version) to every lane.
template <class T>
__device__ __forceinline__ double warp_tree_sum(const T &t, const PwTree &tr, double *val) {
  const int lane = threadIdx.x & 31, grp = lane >> 3;
  for (int base = 0; base < tr.n_leaves; base += 4) {
    const int i = base + grp;
    const bool v = i < tr.n_leaves;
    const double s = leaf_sum8(t, v ? tr.leaf_lo[i] : 0, v ? tr.leaf_n[i] : 0, v);
    if (v && (lane & 7) == 0) val[i] = s;
  }
  __syncwarp();
  int beg = 0;
  for (int h = 0; h < tr.n_levels; ++h) {
    const int end = tr.level_end[h];
    for (int j = beg + lane; j < end; j += 32)
      val[tr.n_leaves + j] = __dadd_rn(val[tr.left[j]], val[tr.right[j]]);
    __syncwarp();
    beg = end;
  }
  const double r = __dadd_rn(0.0, val[tr.n_leaves + beg - 1 < tr.n_leaves ? 0 : tr.n_leaves + beg - 1]);
  __syncwarp();
  return r;
}

// Same sum, lower latency: a lane evaluates all its leaves (g, g + 4, ...)
// with their chains interleaved, so the float64 adds of different leaves
// overlap; the tree itself (tr) should live in shared memory.
constexpr int kPwPerGroup = (kPwMaxLeaves + 3) / 4;
template <class T>
__device__ __forceinline__ double warp_tree_sum_ilp(const T &t, const PwTree &tr, double *val) {
  const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
  const int nl = tr.n_leaves;
  const int per = (nl + 3) / 4;  // leaves per group, warp-uniform bound
  int lo[kPwPerGroup], stop[kPwPerGroup];
  double r[kPwPerGroup];
#pragma unroll
  for (int l = 0; l < kPwPerGroup; ++l) {
    const bool v = g + 4 * l < nl;
    const int m = v ? tr.leaf_n[g + 4 * l] : 0;
    lo[l] = v ? tr.leaf_lo[g + 4 * l] : 0;
    stop[l] = m - m % 8;
    r[l] = 0.0;  // 0.0 + a[j] == a[j] for the non-negative terms here
  }
  // branch-free: every lane issues every load (clamped address), a skipped
  // term adds 0.0, so all chains of a lane overlap
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#pragma unroll
    for (int l = 0; l < kPwPerGroup; ++l) {
      if (l >= per) break;
      const bool ok = 8 * i < stop[l];
      const double v = t.map(t.load(ok ? lo[l] + 8 * i + j : 0));
      r[l] = __dadd_rn(r[l], ok ? v : 0.0);
    }
  }
#pragma unroll
  for (int l = 0; l < kPwPerGroup; ++l) {
    if (l >= per) break;
    const double a = __dadd_rn(r[l], __shfl_down_sync(0xffffffffu, r[l], 1, 8));
    const double b = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, 2, 8));
    double c = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, 4, 8));
    if (g + 4 * l < nl && j == 0) {
      const int m = tr.leaf_n[g + 4 * l];
      if (m < 8) c = 0.0;
      for (int q = stop[l]; q < m; ++q) c = __dadd_rn(c, t.map(t.load(lo[l] + q)));
      val[g + 4 * l] = c;
    }
  }
  __syncwarp();
  int beg = 0;
  for (int h = 0; h < tr.n_levels; ++h) {
    const int end = tr.level_end[h];
    for (int q = beg + lane; q < end; q += 32) val[nl + q] = __dadd_rn(val[tr.left[q]], val[tr.right[q]]);
    __syncwarp();
    beg = end;
  }
  const double res = __dadd_rn(0.0, val[beg == 0 ? 0 : nl + beg - 1]);
  __syncwarp();
  return res;
}

// The same tree sum by the first W warps of the block (threads [0, 32W)),
// synchronised by named barrier `bar` (not 0): 4W groups of 8 lanes share
// the leaves, each group's leaves interleaved.
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
template <int W, class T>
__device__ __noinline__ double group_tree_sum(const T &t, const PwTree &tr, double *val, int bar) {
  constexpr int G = 4 * W;                          // 8-lane groups
  constexpr int PER = (kPwMaxLeaves + G - 1) / G;   // leaves per group (max)
  const int tid = threadIdx.x, g = tid >> 3, j = tid & 7;
  const int nl = tr.n_leaves;
  const int per = (nl + G - 1) / G;
  int lo[PER], stop[PER];
  double r[PER];
#pragma unroll
  for (int l = 0; l < PER; ++l) {
    const bool v = g + G * l < nl;
    const int m = v ? tr.leaf_n[g + G * l] : 0;
    lo[l] = v ? tr.leaf_lo[g + G * l] : 0;
    stop[l] = m - m % 8;
    r[l] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#pragma unroll
    for (int l = 0; l < PER; ++l) {
      if (l >= per) break;
      const bool ok = 8 * i < stop[l];
      const double v = t.map(t.load(ok ? lo[l] + 8 * i + j : 0));
      r[l] = __dadd_rn(r[l], ok ? v : 0.0);
    }
  }
#pragma unroll
  for (int l = 0; l < PER; ++l) {
    if (l >= per) break;
    const double a = __dadd_rn(r[l], __shfl_down_sync(0xffffffffu, r[l], 1, 8));
    const double b = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, 2, 8));
    double c = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, 4, 8));
    if (g + G * l < nl && j == 0) {
      const int m = tr.leaf_n[g + G * l];
      if (m < 8) c = 0.0;
      for (int q = stop[l]; q < m; ++q) c = __dadd_rn(c, t.map(t.load(lo[l] + q)));
      val[g + G * l] = c;
    }
  }
  named_bar(bar, 32 * W);
  int beg = 0;
  for (int h = 0; h < tr.n_levels; ++h) {
    const int end = tr.level_end[h];
    for (int q = beg + tid; q < end; q += 32 * W) val[nl + q] = __dadd_rn(val[tr.left[q]], val[tr.right[q]]);
    named_bar(bar, 32 * W);
    beg = end;
  }
  const double res = __dadd_rn(0.0, val[beg == 0 ? 0 : nl + beg - 1]);
  named_bar(bar, 32 * W);
  return res;
}

// Mean / population variance by the first W warps (see warp_mean_var).
template <int W>
__device__ __noinline__ void group_mean_var(const double *S, int n, const PwTree &tr, double *val,
                                               double *s_part, int bar, double &mean, double &var) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double p0 = 0.0, p1 = 0.0;  // any order: exact below 2^29
  int c = tid;
  for (; c + 32 * W < n; c += 64 * W) {
    p0 = __dadd_rn(p0, S[c]);
    p1 = __dadd_rn(p1, S[c + 32 * W]);
  }
  if (c < n) p0 = __dadd_rn(p0, S[c]);
  double part = __dadd_rn(p0, p1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
  if (lane == 0) s_part[wid] = part;
  named_bar(bar, 32 * W);
  double total = 0.0;
#pragma unroll
  for (int w = 0; w < W; ++w) total = __dadd_rn(total, s_part[w]);
  Term<true> t{S, 0.0, false};
  if (!(total < 536870912.0)) total = group_tree_sum<W>(t, tr, val, bar);
  mean = __ddiv_rn(__dadd_rn(0.0, total), static_cast<double>(n));
  t.mean = mean;
  t.squared = true;
  var = __ddiv_rn(group_tree_sum<W>(t, tr, val, bar), static_cast<double>(n));
}

// Mean and population variance of S[0, n) exactly as numpy (codec.py:299-301)
// by warp 0.  When the any-order float64 total stays below 2^29 every partial
// sum of the pairwise tree is exact (non-negative multiples of 2^-24 below
// 2^29), so the tree equals this plain warp reduction; otherwise the tree
// is evaluated.  The variance terms are rounded, so they always follow the
// tree.
__device__ __forceinline__ void warp_mean_var(const double *S, int n, const PwTree &tr, double *val,
                                              double &mean, double &var) {
  const int lane = threadIdx.x & 31;
  double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;  // any order: exact below 2^29
  int c = lane;
  for (; c + 96 < n; c += 128) {
    p0 = __dadd_rn(p0, S[c]);
    p1 = __dadd_rn(p1, S[c + 32]);
    p2 = __dadd_rn(p2, S[c + 64]);
    p3 = __dadd_rn(p3, S[c + 96]);
  }
  for (; c < n; c += 32) p0 = __dadd_rn(p0, S[c]);
  double part = __dadd_rn(__dadd_rn(p0, p1), __dadd_rn(p2, p3));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
  Term<true> t{S, 0.0, false};
  const double total = part < 536870912.0 ? part : warp_tree_sum_ilp(t, tr, val);
  mean = __ddiv_rn(__dadd_rn(0.0, total), static_cast<double>(n));
  t.mean = mean;
  t.squared = true;
  var = __ddiv_rn(warp_tree_sum_ilp(t, tr, val), static_cast<double>(n));
}

// Flags / ranks / indices for cols <= 8 * blockDim.x with mean, sigma and
// 1/sigma given (same decision rule as outlier_flags_block), one block
// barrier.  s_tmp: 2 * 32 ints of shared memory.  The caller synchronises
// before reading flag / idx.
__device__ __forceinline__ int outlier_flags_fast(const double *S, int64_t rows, int cols,
                                                  double mean, double sigma, double rsig,
                                                  double thr, int64_t k_cap, uint8_t *flag,
                                                  uint32_t *idx, int32_t *k_out, uint32_t *err,
                                                  int *s_tmp, bool too_many_check = true) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int run = (cols + blockDim.x - 1) / blockDim.x;  // <= 32
  const int c0 = min(cols, run * tid), c1 = min(cols, c0 + run);
  const double cap = 65504.0 * static_cast<double>(rows);
  uint32_t f8 = 0;
  int bad = 0;
  for (int base = c0; base < c1; base += 8) {
    uint32_t fb = 0, amb = 0;
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = base + q < c1 ? S[base + q] : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double qa = __dmul_rn(__dsub_rn(v[q], mean), rsig);
      const double margin = __dadd_rn(__dmul_rn(fabs(qa), 0x1p-46), 0x1p-1000);
      const bool hi = qa > __dadd_rn(thr, margin), lo = qa < __dsub_rn(thr, margin);
      const bool live = base + q < c1;
      bad |= live && !(v[q] <= cap);
      fb |= (live && hi && sigma != 0.0 ? 1u : 0u) << q;
      amb |= (live && !hi && !lo && sigma != 0.0 ? 1u : 0u) << q;
    }
    while (amb) {  // rare: within 2^-46 of the threshold (or NaN)
      const int q = __ffs(amb) - 1;
      amb &= amb - 1;
      fb |= (__ddiv_rn(__dsub_rn(v[q], mean), sigma) > thr ? 1u : 0u) << q;
    }
    f8 |= fb << (base - c0);
  }
  // exclusive prefix of the per-thread counts: warp scan + one block barrier
  const int mine = __popc(f8);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const int wbad = __any_sync(0xffffffffu, bad);
  if (lane == 31) {
    s_tmp[wid] = incl;
    s_tmp[32 + wid] = wbad;
  }
  __syncthreads();
  int before = 0, total = 0, anybad = 0;
  for (int w = 0; w < nw; ++w) {
    const int cw = s_tmp[w];
    before += w < wid ? cw : 0;
    total += cw;
    anybad |= s_tmp[32 + w];
  }
  int pos = before + incl - mine;
  uint32_t kept = f8;
  for (uint32_t m = f8; m; m &= m - 1, ++pos) {
    const int q = __ffs(m) - 1;
    if (pos < k_cap) {
      if (idx) idx[pos] = static_cast<uint32_t>(c0 + q);
    } else {
      kept &= ~(1u << q);
    }
  }
  for (int c = c0; c < c1; ++c) flag[c] = static_cast<uint8_t>((kept >> (c - c0)) & 1u);
  if (tid == 0) {
    if (k_out) *k_out = total;
    if (err) {
      if (anybad) atomicOr(err, ADC_ERR_NONFINITE);
      if (too_many_check && 2 * static_cast<int64_t>(total) > cols) atomicOr(err, ADC_ERR_TOO_MANY_OUTLIERS);
      if (total > k_cap) atomicOr(err, ADC_ERR_K_CAP);
    }
  }
  return total;
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
                                                   bool too_many_check) {
  __shared__ int s_tmp[32];
  t.mean = mean;
  t.squared = false;
  const double sigma = __dsqrt_rn(var);
  const double cap = 65504.0 * static_cast<double>(rows);
  // z-score flag (strict >, codec.py:305); a sum above rows * 65504 means an
  // inf/NaN input (no finite f16 matrix reaches it)
  // fl(d / sigma) > thr decided from d * (1/sigma) (relative error < 2^-51
  // against the correctly rounded quotient) unless it lands within 2^-46 of
  // thr; only those few columns pay for the correctly rounded division.
  // Branch-free over a batch of 8 so the float64 latencies overlap.
  const double rsig = sigma != 0.0 ? __drcp_rn(sigma) : 0.0;
  auto z_exact = [&](double v) -> uint32_t {
    return (sigma != 0.0 && __ddiv_rn(__dsub_rn(v, mean), sigma) > thr) ? 1u : 0u;
  };
  const int64_t run = (cols + blockDim.x - 1) / blockDim.x;
  const int64_t c0 = min(cols, run * threadIdx.x), c1 = min(cols, c0 + run);
  int bad = 0, mine = 0, total, pos;
  if (run <= 64) {
    // each thread owns a contiguous run of <= 64 columns: flags in a register mask
    uint64_t bits = 0;
    for (int64_t base = c0; base < c1; base += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = base + q < c1 ? t.load(base + q) : 0.0;
      uint32_t f8 = 0, amb = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double qa = __dmul_rn(__dsub_rn(v[q], mean), rsig);
        const double margin = __dadd_rn(__dmul_rn(fabs(qa), 0x1p-46), 0x1p-1000);
        const bool hi = qa > __dadd_rn(thr, margin), lo = qa < __dsub_rn(thr, margin);
        const bool live = base + q < c1;
        bad |= live && !(v[q] <= cap);
        f8 |= (live && hi && sigma != 0.0 ? 1u : 0u) << q;
        amb |= (live && !hi && !lo && sigma != 0.0 ? 1u : 0u) << q;
      }
      while (amb) {  // rare: within 2^-46 of the threshold (or NaN)
        const int q = __ffs(amb) - 1;
        amb &= amb - 1;
        f8 |= z_exact(v[q]) << q;
      }
      bits |= static_cast<uint64_t>(f8) << (base - c0);
    }
    bad = __syncthreads_or(bad);
    mine = __popcll(bits);
    pos = block_excl_scan(mine, &total, s_tmp);
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
                                           unsigned char *scratch) {
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
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) part = __dadd_rn(part, t.load(c));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
    if ((threadIdx.x & 31) == 0) val[threadIdx.x >> 5] = part;
    __syncthreads();
    double total = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) total = __dadd_rn(total, val[w]);
    __syncthreads();
    if (!(total < 536870912.0)) total = heap_sum(t, n, D, val);
    mean = __ddiv_rn(__dadd_rn(0.0, total), static_cast<double>(cols));
    t.mean = mean;
    t.squared = true;
    var = __ddiv_rn(heap_sum(t, n, D, val), static_cast<double>(cols));
  } else {
    const int depth = build_tree(n, tr, s_lvl, s_tmp);
    mean = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
    t.mean = mean;
    t.squared = true;
    var = __ddiv_rn(tree_sum(t, tr, depth, s_lvl), static_cast<double>(cols));
  }
  return outlier_flags_block(t, mean, var, rows, cols, thr, k_cap, flag, idx, k_out, err,
                             too_many_check);
}

}  // namespace adc
