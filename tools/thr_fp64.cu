// FP64 / FP32 / LDS throughput per SM (one CTA of 512 threads, 8 independent chains per thread)
#include <cstdio>
__global__ void k(double *out, long long *cyc, double a, int n) {
  double x[8]; float f[8];
  for (int i = 0; i < 8; ++i) { x[i] = a + i; f[i] = (float)a + i; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(x[i], a);
  __syncthreads();
  long long t1 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __fadd_rn(f[i], (float)a);
  __syncthreads();
  long long t2 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dmul_rn(x[i], a);
  __syncthreads();
  long long t3 = clock64();
  double s = 0; float g = 0;
  for (int i = 0; i < 8; ++i) { s += x[i]; g += f[i]; }
  out[threadIdx.x] = s + g;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
  const int n = 1000;
  for (int th : {32, 128, 512}) {
    k<<<1, th>>>(o, c, 1.0000001, n); k<<<1, th>>>(o, c, 1.0000001, n);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    double ops = (double)th * 8 * n;
    printf("threads %d: DADD %.2f lanes/clk, FADD %.2f lanes/clk, DMUL %.2f lanes/clk per SM\n", th, ops / h[0], ops / h[1], ops / h[2]);
  }
}
