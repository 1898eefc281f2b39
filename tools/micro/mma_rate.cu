// tcgen05.mma kind::f16 issue/execution rate on B200 as a function of N: one CTA per SM,
// one elected thread issues `reps` batches of 6 MMAs (M = 128, K = 16; the 3-product
// pattern over two accumulators, as variance_f16_kernel issues per 16-point chunk), one
// commit per batch, waits at the end. Operands are zeroed shared memory. Prints cycles
// per MMA and the fraction of the dense FP16 rate (3868 MAC/clk/SM at 2.25 PF, 1.965 GHz),
// and the same for a CTA pair (cta_group::2, M = 256, each CTA holding N/2 rows of B).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mma_rate mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {  // K-major, no swizzle, LBO 128, SBO 256
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

template <int PAIR>
__global__ void __launch_bounds__(128, 1) k(long long* out, int reps, int n, int pattern) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 64);
  unsigned char* A = sm + 1024;          // hi + lo: 2 x 4 KB
  unsigned char* B = sm + 1024 + 8192;   // hi + lo: 2 x 8 KB
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (8192 + 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(A)[i] = 0u;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[0])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (warp == 0 && rank == 0) {
    const uint32_t M = PAIR ? 256u : 128u;
    const uint64_t ah = desc(su32(A)), al = desc(su32(A + 4096)), bh = desc(su32(B)), bl = desc(su32(B + 8192));
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      int nn = n;
      if (pattern == 1) nn = 256 - 16 * (r & 15);  // a triangle pass: N = 256, 240, ..., 16
      if (PAIR && (nn & 31)) nn = (nn + 31) & ~31;
      const uint32_t idesc = (1u << 4) | ((uint32_t)(nn >> 3) << 17) | ((M >> 4) << 24);
      const uint32_t d1 = tmem + 256;
      if (PAIR)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %4, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %5, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %3, %4, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%1], %2, %4, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%1], %2, %5, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%1], %3, %4, %6, 1;\n\t}" ::"r"(tmem),
            "r"(d1), "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc)
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %5, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %4, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %5, %6, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, 1;\n\t}" ::"r"(tmem),
            "r"(d1), "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc)
            : "memory");
    }
    if (PAIR)
      asm volatile(
          "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
              su32(&bars[0]))
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bars[0]))
          : "memory");
    while (!try_wait(su32(&bars[0]), 0)) {
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  } else if (PAIR && warp == 0) {
    while (!try_wait(su32(&bars[0]), 0)) {
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if (warp == 0) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  long long* out;
  cudaMalloc(&out, 148 * sizeof(long long));
  const int smem = 1024 + 8192 + 16384 + 1024;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 4096;
  for (int pair = 0; pair < 2; ++pair)
    for (int pattern = 0; pattern < 2; ++pattern)
      for (int n : {16, 32, 64, 96, 128, 192, 256}) {
        if (pattern == 1 && n != 256) continue;
        if (pair && n < 32) continue;
        long long h[148] = {};
        if (pair) {
          cudaLaunchConfig_t c = {};
          c.gridDim = dim3(148);
          c.blockDim = dim3(128);
          c.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = 2;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          c.attrs = at;
          c.numAttrs = 1;
          cudaLaunchKernelEx(&c, k<1>, out, reps, n, pattern);
        } else {
          k<0><<<148, 128, smem>>>(out, reps, n, pattern);
        }
        const cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        double avg_n = n;
        if (pattern == 1) avg_n = 136.0;
        const double per = (double)mx / (reps * 6.0);
        // per-SM MACs of one MMA: 128 rows x N x 16 (a pair MMA: each SM 128 rows x N)
        const double ideal = 128.0 * avg_n * 16.0 / 3868.0;
        printf("%s %-9s N=%3d: %7.1f cyc/MMA (ideal %6.1f) -> %5.1f%% of dense  [%s]\n", pair ? "pair  " : "single",
               pattern ? "triangle" : "uniform", pattern ? 0 : n, per, ideal, 100.0 * ideal / per,
               cudaGetErrorString(e));
      }
  return 0;
}
