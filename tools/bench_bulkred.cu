// Microbenchmark: cross-CTA column-sum reduction options on B200.
//   (1) cp.reduce.async.bulk .add.f64 (UBLKRED) of a cols-double smem array
//       from every CTA into one global array;
//   (2) one red.global.add.f64 per column per CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_bulkred.bin tools/bench_bulkred.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k_bulk(double *g, int cols, int reps) {
  extern __shared__ __align__(128) double s[];
  for (int c = threadIdx.x; c < cols; c += blockDim.x) s[c] = 1.0 + c;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r = 0; r < reps; ++r) {
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(g),
                   "r"((unsigned)__cvta_generic_to_shared(s)), "r"(cols * 8)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void __launch_bounds__(1024, 1) k_red(double *g, int cols, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int c = threadIdx.x; c < cols; c += blockDim.x)
      asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(g + c), "d"(1.0 + c) : "memory");
}
__global__ void __launch_bounds__(1024, 1) k_empty(double *g, int cols, int reps) {}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *g;
  cudaMalloc(&g, 16384 * 8);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int cols : {1024, 4096, 11008}) {
    for (int kind = 0; kind < 3; ++kind) {
      auto kern = kind == 0 ? k_bulk : kind == 1 ? k_red : k_empty;
      for (int w = 0; w < 3; ++w) kern<<<sms, 1024, cols * 8>>>(g, cols, 1);
      cudaEventRecord(a);
      const int it = 50;
      for (int i = 0; i < it; ++i) kern<<<sms, 1024, cols * 8>>>(g, cols, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("cols %5d %-10s %7.2f us/launch\n", cols, kind == 0 ? "bulk-red" : kind == 1 ? "red.f64" : "empty",
             ms * 1e3 / it);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
