// Latency / throughput probe for the float64 ops the column statistics use.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double *out, long long *cyc, double a, int n) {
  double x = a, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  long long t1 = clock64();
  float f = (float)a, g = f * 0.5f;
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, g);
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = __ddiv_rn(z, 1.0000001);
  long long t3 = clock64();
  int k = (int)a;
  for (int i = 0; i < n; ++i) k = __shfl_xor_sync(0xffffffffu, k, 1) + 1;
  long long t4 = clock64();
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = a;
  __syncthreads();
  long long t5 = clock64();
  double w = 0; int p = threadIdx.x & 63;
  for (int i = 0; i < n; ++i) { w = __dadd_rn(w, sm[p]); p = (p + (int)w) & 63; }
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    out[0] = x + f + z + k + w;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t6 - t5; cyc[5] = t7 - t6;
  }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  const int n = 1000;
  for (int threads : {32, 256}) {
    chain<<<1, threads>>>(o, c, 1.5, n);
    chain<<<1, threads>>>(o, c, 1.5, n);
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("threads %d: per-op cycles  dadd %.1f  fadd %.1f  ddiv %.1f  shfl+iadd %.1f  lds+dadd %.1f  bar %.1f\n", threads,
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
  }
  return 0;
}
