// Microbenchmark: tcgen05.commit -> mbarrier arrive latency, with 0 / 1 / 6 TF32 MMAs
// (M=128, N=256, K=8, operands from zeroed shared memory) in flight, and the
// cp.async.bulk completion latency of a 32 KB L2-resident block.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o commit_latency commit_latency.cu
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
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) |
         (1ull << 46);
}

__global__ void __launch_bounds__(128, 1) k(const float* gsrc, long long* out, int iters, int nmma) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 64);
  float* A = reinterpret_cast<float*>(sm + 1024);          // 128 x 8 tf32, 4 KB
  float* B = reinterpret_cast<float*>(sm + 1024 + 4096);   // 256 x 8 tf32, 8 KB
  float* C = reinterpret_cast<float*>(sm + 1024 + 12288);  // 32 KB bulk-copy target
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 1024 + 2048; i += blockDim.x) A[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t da = desc(su32(A), 256), db = desc(su32(B), 256);
    uint32_t ph = 0;
    long long tot = 0;
    for (int it = 0; it < iters; ++it) {
      const long long t0 = clock64();
      for (int m = 0; m < nmma; ++m)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc)
            : "memory");
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bars[0])) : "memory");
      while (!try_wait(su32(&bars[0]), ph)) {
      }
      ph ^= 1u;
      tot += clock64() - t0;
    }
    if (threadIdx.x == 0) out[nmma == 0 ? 0 : nmma == 1 ? 1 : 2] = tot / iters;
    // bulk copy latency, 32 KB
    if (nmma == 0) {
      uint32_t ph1 = 0;
      long long tb = 0;
      for (int it = 0; it < iters; ++it) {
        const long long t0 = clock64();
        if (threadIdx.x == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[1])), "r"(32768u) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(C)),
                       "l"(gsrc), "r"(32768u), "r"(su32(&bars[1]))
                       : "memory");
        }
        while (!try_wait(su32(&bars[1]), ph1)) {
        }
        ph1 ^= 1u;
        tb += clock64() - t0;
      }
      if (threadIdx.x == 0) out[3] = tb / iters;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  float* src;
  long long* out;
  cudaMalloc(&src, 1 << 20);
  cudaMemset(src, 0, 1 << 20);
  cudaMalloc(&out, 64);
  const int smem = 1024 + 12288 + 32768 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[4];
  for (int nm : {0, 1, 6}) k<<<1, 128, smem>>>(src, out, 200, nm);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
  printf("%s commit->wait: 0 MMA %lld cyc, 1 MMA %lld cyc, 6 MMA %lld cyc; 32KB bulk copy %lld cyc\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
  return 0;
}
