// Microbenchmark: dependent-chain latencies on this GPU (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed, int n) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);           // DFMA chain
  long long t1 = clock64();
  double s = x;
  for (int i = 0; i < n; ++i) s += __shfl_xor_sync(0xffffffffu, s, 1) * 1e-300;  // SHFL+DADD chain
  long long t2 = clock64();
  double d = x;
  for (int i = 0; i < n; ++i) d = 1.0 / (d + 1.0);             // DDIV chain
  long long t3 = clock64();
  double e = -0.5;
  for (int i = 0; i < n; ++i) e = -exp(e) * 0.5;               // libm exp chain
  long long t4 = clock64();
  float f = x;
  for (int i = 0; i < n; ++i) f = fmaf(f, 1.0000001f, 1e-12f); // FFMA chain
  long long t5 = clock64();
  out[threadIdx.x] = x + s + d + e + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
__global__ void bar(long long* cyc, int n) {
  __shared__ double s[32];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { if (threadIdx.x == 0) s[0] += 1.0; __syncthreads(); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 8);
  const int n = 4096;
  k<<<1, 32>>>(o, c, 0.5, n); bar<<<1, 128>>>(c, n); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  printf("DFMA %.1f  SHFL+DMUL+DADD %.1f  DDIV %.1f  exp %.1f  FFMA %.1f  syncthreads(128t,+STS) %.1f cycles\n",
         h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
  return 0;
}
