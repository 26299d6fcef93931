// Delivery rate of a 148-CTA slab read from HBM, the access pattern of the
// single-pass outlier kernel's phase A (k4.cu): every CTA reads its own
// contiguous slab (bytes_per_cta) either with 1-D TMA bulk copies of `chunk`
// bytes (all issued up front, one mbarrier each) or with plain 16-byte loads
// (each thread `depth` loads in flight), into shared memory.  Buffers rotate
// through 2 GB so every launch streams from HBM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_stream.bin tools/bench_stream.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(512, 1) tma_slab(const char *src, int bytes_per_cta, int chunk, unsigned *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const int n = bytes_per_cta / chunk;
  const char *s = src + static_cast<long long>(blockIdx.x) * bytes_per_cta;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int i = 0; i < n; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[i])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(sm + i * chunk)), "l"(s + static_cast<long long>(i) * chunk), "r"(chunk), "r"(sa(&bar[i]))
                   : "memory");
    }
  }
  __syncthreads();
  unsigned acc = 0;
  for (int i = 0; i < n; ++i) {
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}"
                 ::"r"(sa(&bar[i])) : "memory");
    acc += reinterpret_cast<const unsigned *>(sm + i * chunk)[threadIdx.x];
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void __launch_bounds__(512, 1) ldg_slab(const uint4 *src, int bytes_per_cta, unsigned *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int n16 = bytes_per_cta / 16;
  const uint4 *s = src + static_cast<long long>(blockIdx.x) * n16;
  uint4 *d = reinterpret_cast<uint4 *>(sm);
  constexpr int D = 8;
  for (int i = threadIdx.x; i < n16; i += 512 * D) {
    uint4 v[D];
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (i + j * 512 < n16) v[j] = __ldcs(s + i + j * 512);
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (i + j * 512 < n16) d[i + j * 512] = v[j];
  }
  __syncthreads();
  if (reinterpret_cast<unsigned *>(sm)[threadIdx.x] == 0x12345678u) *sink = 1;
}

int main() {
  const long long total = 2ll << 30;
  char *src;
  unsigned *sink;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(tma_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(ldg_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  for (int per : {113 * 1024, 192 * 1024}) {
    const long long per_launch = 148ll * per;
    const int nbuf = static_cast<int>(total / per_launch);
    for (int chunk : {16384, 32768, 0}) {
      if (chunk && per % chunk) continue;
      for (int w = 0; w < 2; ++w) {
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) {
          const char *p = src + (r % nbuf) * per_launch;
          if (chunk) tma_slab<<<148, 512, 200 * 1024>>>(p, per, chunk, sink);
          else ldg_slab<<<148, 512, 200 * 1024>>>(reinterpret_cast<const uint4 *>(p), per, sink);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      printf("slab %3d KB/CTA %-10s chunk %6d: %6.2f us per launch, %6.0f GB/s\n", per / 1024, chunk ? "TMA" : "LDG+STS",
             chunk, us, per_launch / us / 1e3);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
