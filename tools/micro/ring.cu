// Cost of an empty producer/consumer mbarrier ring like the variance kernels': S stages,
// P producer warps (lane 0 waits on empty[s], the warp arrives on full[s]), one consumer
// warp (waits on full[s], frees the stage with tcgen05.commit -> empty[s], or with a plain
// mbarrier arrive). No work per stage. Prints cycles per stage.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ring ring.cu
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
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__global__ void ring(long long* out, int iters, int S, int P, int use_commit) {
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(P));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const long long t0 = clock64();
  if (warp == 0) {  // consumer
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      while (!try_wait(su32(&full[s]), ph)) {
      }
      if (use_commit)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&empty[s]))
            : "memory");
      else if (lane == 0)
        arrive(su32(&empty[s]));
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (lane == 0) out[0] = (clock64() - t0) / iters;
  } else if (warp <= P) {  // producers
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      if (lane == 0)
        while (!try_wait(su32(&empty[s]), ph ^ 1u)) {
        }
      __syncwarp();
      if (lane == 0) arrive(su32(&full[s]));
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}

int main() {
  long long* out;
  cudaMalloc(&out, 8);
  for (int commit = 0; commit < 2; ++commit)
    for (int P : {1, 8})
      for (int S : {3, 4, 8}) {
        ring<<<148, 32 * (P + 1)>>>(out, 20000, S, P, commit);
        const cudaError_t e = cudaDeviceSynchronize();
        long long h = 0;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("%-13s producers %d stages %d: %lld cycles per stage [%s]\n", commit ? "tcgen05.commit" : "mbarrier.arrive",
               P, S, h, cudaGetErrorString(e));
      }
  return 0;
}
