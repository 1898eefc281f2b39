// Measured FP64 FMA (DFMA) and FP32 FFMA throughput of the whole GPU: the denominator
// of the rollout kernel's roofline (its binding pipe is FP64).
// 8 independent FMA chains per thread, 4 blocks of 256 threads per SM, CUDA events,
// best of 5. Prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <class T>
__global__ void __launch_bounds__(256) fma_chains(T* out, T a, T b, int iters) {
  T x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = a + (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], b, a);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == (T)12345.678) out[threadIdx.x] = s;  // keeps the chains live
}

template <class T>
double run(int sms, int iters) {
  T* d = nullptr;
  cudaMalloc(&d, 256 * sizeof(T));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4;
  fma_chains<T><<<blocks, 256>>>(d, (T)0.5, (T)0.999, iters);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_chains<T><<<blocks, 256>>>(d, (T)0.5, (T)0.999, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(d);
  const double flop = 2.0 * 8.0 * (double)iters * blocks * 256;
  return flop / (best * 1e-3) / 1e12;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double f64 = run<double>(sms, 1 << 14);
  const double f32 = run<float>(sms, 1 << 16);
  printf("{\"fp64_fma_tflops\": %.3f, \"fp32_fma_tflops\": %.3f, \"sms\": %d, \"clock_khz\": %d, "
         "\"how\": \"8 independent FMA chains/thread, 4x256-thread blocks per SM, best of 5, CUDA events\"}\n",
         f64, f32, sms, clk);
  return 0;
}
