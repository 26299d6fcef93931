// Sub-step timing of warp_mean_var / outlier_flags_fast (one CTA, 512 threads).
#include <cstdio>
#ifndef REPS_DEV
#define REPS_DEV 1
#endif
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
__global__ void __launch_bounds__(512) k(const double *Sg, int n, PwTree tr, long long *cyc, double *out) {
  __shared__ double S[4096];
  __shared__ double val[600];
  __shared__ uint8_t flag[4104];
  __shared__ uint32_t sidx[4096];
  __shared__ double ms[3];
  __shared__ PwTree st;
  __shared__ int s_tmp[64];
  if (threadIdx.x == 0) st = tr;
  for (int c = threadIdx.x; c < n; c += blockDim.x) S[c] = Sg[c];
  __syncthreads();
  long long c0 = clock64(), c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double mean, var0;
    warp_mean_var(S, n, st, val, mean, var0);
    c1 = clock64();
    c2 = clock64();
    Term<true> t{S, mean, true};
    double s2 = 0;
    const int reps = REPS_DEV;
    for (int rr = 0; rr < reps; ++rr) { s2 += warp_tree_sum_ilp(t, st, val); t.mean += 1e-300; }
    c3 = clock64();
    const double var = __ddiv_rn(s2, (double)n);
    const double sigma = __dsqrt_rn(var);
    const double rs = __drcp_rn(sigma);
    c4 = clock64();
    if (lane == 0) { ms[0] = mean; ms[1] = sigma; ms[2] = rs; }
  }
  __syncthreads();
  long long d0 = clock64();
  int kk = outlier_flags_fast(S, 8192, n, ms[0], ms[1], ms[2], 3.0, n, flag, sidx, nullptr, nullptr, s_tmp);
  __syncthreads();
  c5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - d0; out[0] = ms[0]; out[1] = ms[1]; out[2] = kk; }
}
int main() {
  for (int n : {1024, 4096}) {
    std::vector<double> h(n);
    for (int i = 0; i < n; ++i) h[i] = 1000.0 + (i * 7919 % 1000) * 0.375 + (i % 97 == 0 ? 40000 : 0);
    double *Sg, *out; long long *cyc;
    cudaMalloc(&Sg, n * 8); cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
    cudaMemcpy(Sg, h.data(), n * 8, cudaMemcpyHostToDevice);
    PwTree tr; build(n, tr);
    for (int r = 0; r < 3; ++r) k<<<1, 512>>>(Sg, n, tr, cyc, out);
    long long c[5]; double o[3];
    cudaMemcpy(c, cyc, 40, cudaMemcpyDeviceToHost); cudaMemcpy(o, out, 24, cudaMemcpyDeviceToHost);
    printf("n=%d: lane sums %lld, shfl-reduce+div %lld, var tree %lld, div+sqrt+rcp %lld, flags %lld cycles | mean %.17g sigma %.17g k %g (%s)\n",
           n, c[0], c[1], c[2], c[3], c[4], o[0], o[1], o[2], cudaGetErrorString(cudaGetLastError()));
  }
}
