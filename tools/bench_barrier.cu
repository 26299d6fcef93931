// Microbenchmark: cross-CTA reduction + grid barrier costs on one B200
// (design input for fused.cu).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -o /tmp/bb tools/bench_barrier.cu && /tmp/bb
// Variants, each timed over ITERS rounds inside one cooperative launch of one
// 512-thread CTA per SM:
//   0  barrier only (atomicAdd arrive + acquire spin, generation counter)
//   1  1024 f64 atomics per CTA into one [1024] array, then barrier
//   2  partials to [P][1024] (plain stores), barrier, column-slice reduce, barrier
//   3  like 1 but red.global (no return) + fence
#include <cstdio>
#include <cuda_runtime.h>

constexpr int T = 512;
constexpr int COLS = 1024;
constexpr int ITERS = 50;

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ void grid_bar(unsigned *cnt, unsigned *gen, unsigned P) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acq(gen);
    __threadfence();
    if (atomicAdd(cnt, 1u) == P - 1) {
      *cnt = 0;
      __threadfence();
      atomicExch(gen, g + 1);
    } else {
      while (ld_acq(gen) == g) {
      }
    }
  }
  __syncthreads();
}

// arrive = red.release (no return value), wait = acquire-poll of a counter
// that only grows within the launch: round r completes at (r + 1) * P.
__device__ void grid_bar2(unsigned *cnt, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    while (ld_acq(cnt) < target) {
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(T, 1) kern(int variant, double *acc, double *part, double *S,
                                             unsigned *cnt, unsigned *gen, long long *out) {
  const unsigned P = gridDim.x;
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    if (variant == 1) {
      for (int c = threadIdx.x; c < COLS; c += T) atomicAdd(acc + c, 1.0);
      grid_bar(cnt, gen, P);
    } else if (variant == 4) {
      grid_bar2(cnt + 16, (it + 1) * P);
    } else if (variant == 5) {
      for (int c = threadIdx.x; c < COLS; c += T)
        asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(acc + c), "d"(1.0) : "memory");
      grid_bar2(cnt + 16, (it + 1) * P);
    } else if (variant == 6) {
      // 8 columns per atomic thread-slot: only 128 threads issue, 8 each
      if (threadIdx.x < COLS / 8)
        for (int j = 0; j < 8; ++j)
          asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(acc + threadIdx.x * 8 + j), "d"(1.0) : "memory");
      grid_bar2(cnt + 16, (it + 1) * P);
    } else if (variant == 3) {
      for (int c = threadIdx.x; c < COLS; c += T)
        asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(acc + c), "d"(1.0) : "memory");
      grid_bar(cnt, gen, P);
    } else if (variant == 2) {
      for (int c = threadIdx.x; c < COLS; c += T) __stcg(part + blockIdx.x * COLS + c, 1.0);
      grid_bar(cnt, gen, P);
      const int c0 = COLS * blockIdx.x / P, c1 = COLS * (blockIdx.x + 1) / P;
      // lanes over partials, warps over columns
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      for (int c = c0 + w; c < c1; c += T / 32) {
        double v = 0;
        for (int b = l; b < P; b += 32) v += __ldcg(part + b * COLS + c);
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (l == 0) __stcg(S + c, v);
      }
      grid_bar(cnt, gen, P);
      double s = 0;
      for (int c = threadIdx.x; c < COLS; c += T) s += __ldcg(S + c);
      if (s < 0) out[1] = 1;
    } else {
      grid_bar(cnt, gen, P);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *acc, *part, *S;
  unsigned *cnt;
  long long *out;
  cudaMalloc(&acc, COLS * 8);
  cudaMalloc(&part, (size_t)sms * COLS * 8);
  cudaMalloc(&S, COLS * 8);
  cudaMalloc(&cnt, 64);
  cudaMalloc(&out, 64);
  cudaMemset(cnt, 0, 64);
  cudaMemset(acc, 0, COLS * 8);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char *names[] = {"barrier only", "f64 atomicAdd x1024 + barrier",
                         "partials + barrier + slice reduce + barrier", "red.f64 x1024 + barrier", "red.release barrier", "red.f64 x1024 + red.release barrier",
                         "red.f64 x1024 (128 thr x 8) + red.release barrier"};
  for (int v = 0; v < 7; ++v) {
    cudaMemset(cnt, 0, 64);
    for (int rep = 0; rep < 2; ++rep) {
      unsigned *gen = cnt + 8;
      void *args[] = {&v, &acc, &part, &S, &cnt, &gen, &out};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel((void *)kern, dim3(sms), dim3(T), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      long long cyc = 0;
      cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
      if (rep)
        printf("%-48s %s: %.3f us/round (clock64), event %.2f us total for %d rounds\n", names[v],
               cudaGetErrorString(e), cyc / (clk / 1e3) / ITERS, ms * 1e3, ITERS);
    }
  }
  // launch latency of an empty cooperative vs normal launch, eager
  for (int coop = 0; coop < 2; ++coop) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int v = 9;
    unsigned *gen = cnt + 8;
    void *args[] = {&v, &acc, &part, &S, &cnt, &gen, &out};
    cudaEventRecord(a);
    for (int i = 0; i < 100; ++i) {
      if (coop)
        cudaLaunchCooperativeKernel((void *)kern, dim3(sms), dim3(T), args, 0, 0);
      else
        cudaLaunchKernel((void *)kern, dim3(sms), dim3(T), args, 0, 0);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s launch of a %d-barrier kernel: %.2f us per launch\n", coop ? "cooperative" : "normal",
           ITERS, ms * 1e3 / 100);
  }
  return 0;
}
