// Isolated cost of the fused kernel's statistics stages (clock64, one CTA of
// 512 threads): warp-0 pairwise tree sums (mean, var) and the block flags.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false
//   --expt-relaxed-constexpr -I paper_2508_00806_b200/csrc -o tools/bench_stats.bin tools/bench_stats.cu
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>
#include <algorithm>
#include "stats.cuh"
using namespace adc;

static bool build(int n, PwTree &t) {
  struct In { int l, r, h; };
  std::vector<In> in; std::vector<std::pair<int,int>> lv;
  std::function<std::pair<int,int>(int,int)> rec = [&](int lo, int m) -> std::pair<int,int> {
    if (m <= 128) { lv.emplace_back(lo, m); return {(int)lv.size() - 1, 0}; }
    int h = m / 2 - (m / 2) % 8; auto a = rec(lo, h), b = rec(lo + h, m - h);
    in.push_back({a.first, b.first, 1 + std::max(a.second, b.second)}); return {-(int)in.size(), in.back().h}; };
  rec(0, n);
  int nl = lv.size(), ni = in.size(); std::vector<int> o(ni), pos(ni);
  for (int i = 0; i < ni; ++i) o[i] = i;
  std::stable_sort(o.begin(), o.end(), [&](int x, int y) { return in[x].h < in[y].h; });
  for (int i = 0; i < ni; ++i) pos[o[i]] = i;
  auto id = [&](int e) { return e >= 0 ? e : nl + pos[-e - 1]; };
  t = PwTree{}; t.n_leaves = nl;
  for (int i = 0; i < nl; ++i) { t.leaf_lo[i] = lv[i].first; t.leaf_n[i] = lv[i].second; }
  int L = 0;
  for (int j = 0; j < ni; ++j) { auto &v = in[o[j]]; t.left[j] = id(v.l); t.right[j] = id(v.r); L = std::max(L, v.h); t.level_end[v.h - 1] = j + 1; }
  t.n_levels = L; return true;
}

__global__ void __launch_bounds__(512) k(const double *Sg, int n, PwTree tr, long long *cyc, double *out, uint8_t *fl, uint32_t *idx, int reps) {
  __shared__ double S[4096];
  __shared__ double val[600];
  __shared__ uint8_t flag[4104];
  __shared__ uint32_t sidx[4096];
  __shared__ double ms[2];
  for (int c = threadIdx.x; c < n; c += blockDim.x) S[c] = Sg[c];
  __syncthreads();
  long long t0 = clock64(), t1 = 0;
  int kk = 0;
  for (int rep = 0; rep < reps; ++rep) {
  if (threadIdx.x < 32) {
    Term<true> t{S, 0.0, false};
    double mean = __ddiv_rn(warp_tree_sum(t, tr, val), (double)n);
    t.mean = mean; t.squared = true;
    double var = __ddiv_rn(warp_tree_sum(t, tr, val), (double)n);
    if (threadIdx.x == 0) { ms[0] = mean; ms[1] = var; }
  }
  __syncthreads();
  t1 = clock64();
  kk += outlier_flags_block(Term<true>{S, 0.0, false}, ms[0], ms[1], 8192, n, 3.0, n, flag, sidx, nullptr, nullptr, true);
  }
  long long t2 = clock64();
  // block heap version for comparison
  double *v2 = val;
  Term<true> t{S, 0.0, false};
  const int D = heap_depth(n);
  double mean2 = __ddiv_rn(heap_sum(t, n, D, v2), (double)n);
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; out[0] = ms[0]; out[1] = ms[1]; out[2] = mean2; out[3] = kk; }
}

int main() {
  for (int n : {768, 1024, 4096}) {
    std::vector<double> h(n);
    for (int i = 0; i < n; ++i) h[i] = 1000.0 + (i * 7919 % 1000) * 0.37 + (i % 97 == 0 ? 40000 : 0);
    double *Sg, *out; long long *cyc; uint8_t *fl; uint32_t *idx;
    cudaMalloc(&Sg, n * 8); cudaMalloc(&out, 64); cudaMalloc(&cyc, 64); cudaMalloc(&fl, n + 8); cudaMalloc(&idx, n * 4);
    cudaMemcpy(Sg, h.data(), n * 8, cudaMemcpyHostToDevice);
    PwTree tr; build(n, tr);
    int reps = getenv("REPS") ? atoi(getenv("REPS")) : 1;
    for (int r = 0; r < 2; ++r) k<<<1, 512>>>(Sg, n, tr, cyc, out, fl, idx, reps);
    long long c[3]; double o[4];
    cudaMemcpy(c, cyc, 24, cudaMemcpyDeviceToHost); cudaMemcpy(o, out, 32, cudaMemcpyDeviceToHost);
    printf("n=%d: warp mean+var %lld cyc, flags %lld cyc, block heap mean %lld cyc | mean %.17g var %.17g heapmean %.17g k %g (%s)\n",
           n, c[0], c[1], c[2], o[0], o[1], o[2], o[3], cudaGetErrorString(cudaGetLastError()));
  }
}
