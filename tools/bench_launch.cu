// Launch-cost microbenchmark: back-to-back launches of persistent-style
// kernels (one CTA per SM) with different shared-memory footprints.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_launch.bin tools/bench_launch.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_empty(int *p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p[0] == 12345) s[0] = 1, p[1] = s[0];
}
__global__ void __launch_bounds__(512, 1) k_touch(int *p, int n) {
  extern __shared__ int s[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = i;
  __syncthreads();
  if (threadIdx.x == 0 && s[n - 1] == 12345) p[1] = 1;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int *p;
  cudaMalloc(&p, 64);
  cudaMemset(p, 0, 64);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_touch, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int kb : {0, 16, 48, 64, 100, 128, 160, 200, 220, 226}) {
    for (int touch = 0; touch < (kb ? 2 : 1); ++touch) {
      size_t sm = kb * 1024;
      for (int w = 0; w < 20; ++w)
        touch ? k_touch<<<sms, 512, sm>>>(p, (int)(sm / 4 > 0 ? sm / 4 : 1)) : k_empty<<<sms, 512, sm>>>(p);
      cudaEventRecord(a);
      const int it = 50;
      for (int i = 0; i < it; ++i)
        touch ? k_touch<<<sms, 512, sm>>>(p, (int)(sm / 4 > 0 ? sm / 4 : 1)) : k_empty<<<sms, 512, sm>>>(p);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("dyn smem %3d KB %-6s %7.2f us/launch\n", kb, touch ? "touch" : "empty", ms * 1e3 / it);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
