// Micro-benchmarks behind the single-pass kernel's design (k4.cu):
//  1. issue cost of cp.async.bulk (TMA) copies from one thread vs their size;
//  2. cold vs warm straight-line code (instruction-cache misses at kernel start);
//  3. per-thread cp.async (LDGSTS) streaming of a 16 KB-per-warp tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_issue.bin tools/bench_issue.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void tma_issue(const char *src, long long *out, int n, int bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const char *s = src + static_cast<long long>(blockIdx.x) * n * bytes;
    long long t0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * bytes) : "memory");
    for (int i = 0; i < n; ++i)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(sm + (i * bytes) % (192 * 1024))), "l"(s + static_cast<long long>(i) * bytes), "r"(bytes),
                   "r"(sa(&bar)) : "memory");
    long long t1 = clock64();
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}"
                 ::"r"(sa(&bar)) : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
}

#define R8(x) x x x x x x x x
#define R64(x) R8(R8(x))
__global__ void code(long long *out, int v) {
  int a = v, b = v + 1, c = v + 2, d = v + 3;
  long long t0 = clock64();
  R64(R8(asm volatile("add.s32 %0, %0, %4; add.s32 %1, %1, %4; add.s32 %2, %2, %4; add.s32 %3, %3, %4;"
                      : "+r"(a), "+r"(b), "+r"(c), "+r"(d) : "r"(v));))
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = a + b + c + d; }
}

template <int depth>
__global__ void ldgsts(const uint4 *src, long long *out, int rows) {
  extern __shared__ __align__(128) unsigned char sm[];
  // thread t copies rows of 32 B (two 16 B pieces) of its own column slot, depth rows ahead
  const int t = threadIdx.x;
  const uint4 *s = src + static_cast<long long>(blockIdx.x) * rows * 1024 + 2 * (t % 64) + (t / 64) * 128;
  long long t0 = clock64();
  unsigned acc = 0;
  for (int r = 0; r < rows; r += 8) {
    const int slot = (r / 8) % depth;
    unsigned char *d = sm + slot * 16384 + 32 * t;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(d)), "l"(s + static_cast<long long>(r) * 128));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(d + 16)), "l"(s + static_cast<long long>(r) * 128 + 1));
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (r / 8 >= depth - 1) {
      asm volatile("cp.async.wait_group %0;" ::"n"(depth - 1) : "memory");
      const int cs = ((r / 8) - (depth - 1)) % depth;
      acc += *reinterpret_cast<const unsigned *>(sm + cs * 16384 + 32 * t);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  if (t == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 0xdeadbeef) out[1] = acc;
}

int main() {
  char *src;
  long long *out, h[2];
  cudaMalloc(&src, 1ll << 30);
  cudaMemset(src, 1, 1ll << 30);
  cudaMalloc(&out, 64);
  cudaFuncSetAttribute(tma_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int bytes : {2048, 16384}) {
    for (int n : {1, 4, 8, 13, 32, 48}) {
      if (static_cast<long long>(n) * bytes >= (1 << 20)) continue;
      for (int rep = 0; rep < 2; ++rep) tma_issue<<<148, 128, 200 * 1024>>>(src, out, n, bytes);
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("TMA %6d B x %3d: issue %7lld cyc (%5.0f/copy), complete %7lld cyc (%.1f GB/s per SM at 1.965 GHz)\n", bytes,
             n, h[0], double(h[0]) / n, h[1], double(n) * bytes / (h[1] / 1.965));
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    code<<<148, 32>>>(out, rep);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("straight-line 2048 IADD (512 x 4 chains), launch %d: %lld cyc\n", rep, h[0]);
  }
  auto run = [&](auto kern, int depth) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<148, 512, depth * 16384>>>(reinterpret_cast<const uint4 *>(src), out, 8 * 256);
    kern<<<148, 512, depth * 16384>>>(reinterpret_cast<const uint4 *>(src), out, 8 * 256);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    const double bytes = 256.0 * 16384;
    (void)0;
    printf("LDGSTS depth %2d: %lld cyc for %.0f KB per SM: %.1f GB/s per SM, %.0f GB/s chip\n", depth, h[0], bytes / 1024,
           bytes / (h[0] / 1.965), 148 * bytes / (h[0] / 1.965));
  };
  run(ldgsts<4>, 4);
  run(ldgsts<8>, 8);
  run(ldgsts<12>, 12);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
