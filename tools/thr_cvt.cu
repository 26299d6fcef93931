// Throughput of the conversions on the exact column-sum path (per SM, one
// CTA of 512 threads, 8 independent chains per thread):
//   F2F.F64.F32, F2F.F64.F16 (cvt to double) and DADD, vs an integer-built
//   double (shift + add on the f32 bits) + DADD.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/thr_cvt.bin tools/thr_cvt.cu
#include <cstdio>
#include <cuda_fp16.h>

__global__ void k(double *out, long long *cyc, float a, int n) {
  double acc[8];
  float f[8];
  __half h[8];
  for (int i = 0; i < 8; ++i) { acc[i] = 0; f[i] = a + i; h[i] = __float2half(a + i); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i] += (double)f[i];
      f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);  // keep the input live and changing
    }
  }
  __syncthreads();
  long long t1 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc[i] += (double)__half2float(h[i]);
      h[i] = __ushort_as_half(__half_as_ushort(h[i]) ^ 1);
    }
  }
  __syncthreads();
  long long t2 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const unsigned b = __float_as_uint(f[i]);
      acc[i] += __hiloint2double(static_cast<int>((b >> 3) + 0x38000000u), 0);
      f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);
    }
  }
  __syncthreads();
  long long t3 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += 1.0;
  }
  __syncthreads();
  long long t4 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i] + f[i] + __half2float(h[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
}

int main() {
  double *out; long long *cyc;
  cudaMalloc(&out, 148 * 512 * sizeof(double));
  cudaMallocManaged(&cyc, 4 * sizeof(long long));
  const int n = 4096;
  k<<<148, 512>>>(out, cyc, 1.5f, n);
  cudaDeviceSynchronize();
  k<<<148, 512>>>(out, cyc, 1.5f, n);
  cudaDeviceSynchronize();
  const double ops = 512.0 * 8 * n;
  const char *names[4] = {"F2F.F64.F32 + DADD", "F2F f16->f32->f64 + DADD", "int-built f64 + DADD", "DADD only"};
  for (int i = 0; i < 4; ++i) printf("%-28s %6.1f elements/clk/SM\n", names[i], ops / cyc[i]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
