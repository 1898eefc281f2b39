// Dependent-chain cost of the heading wrap: remainder()-based vs rint+fma (bit-identical),
// with omega read from shared memory vs from global (L2) scratch.
#include <cstdio>
#include <cuda_runtime.h>
constexpr double kPi = 3.14159265358979323846;
__device__ __forceinline__ double wrap_rem(double a) {
  double r = remainder(a, 2.0 * kPi);
  if (r <= -kPi) r += 2.0 * kPi;
  return r;
}
__device__ __forceinline__ double wrap_fast(double a) {
  const double P = 2.0 * kPi;
  double r;
  if (fabs(a) < 0x1p40) {
    double n = rint(a * (1.0 / (2.0 * kPi)));
    r = fma(-n, P, a);
    if (r > kPi) { n += 1.0; r = fma(-n, P, a); }
    else if (r < -kPi) { n -= 1.0; r = fma(-n, P, a); }
    if (fabs(r) == kPi && ((long long)n & 1)) { n += r > 0.0 ? 1.0 : -1.0; r = fma(-n, P, a); }
    if (r == 0.0) r = copysign(0.0, a);
  } else {
    r = remainder(a, P);
  }
  if (r <= -kPi) r += P;
  return r;
}
__global__ void k(const double* gw, double* out, long long* cyc, int T) {
  __shared__ double sw[64];
  if (threadIdx.x < 64) sw[threadIdx.x] = gw[threadIdx.x];
  __syncthreads();
  double th = 0.3;
  long long t0 = clock64();
  for (int i = 0; i < T; ++i) th = wrap_rem(th + sw[i] * 0.1);
  long long t1 = clock64();
  double th2 = 0.3;
  for (int i = 0; i < T; ++i) th2 = wrap_fast(th2 + sw[i] * 0.1);
  long long t2 = clock64();
  double th3 = 0.3;
  for (int i = 0; i < T; ++i) th3 = wrap_rem(th3 + gw[64 + i] * 0.1);
  long long t3 = clock64();
  double th4 = 0.3;
  for (int i = 0; i < T; ++i) th4 = wrap_fast(th4 + gw[128 + i] * 0.1);
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = th + th2 + th3 + th4;
}
int main() {
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 3.0 * ((i * 37) % 11 - 5);
  double *gw, *out; long long* cyc;
  cudaMalloc(&gw, sizeof h); cudaMalloc(&out, 1024); cudaMallocManaged(&cyc, 64);
  cudaMemcpy(gw, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(gw, out, cyc, 40);
  cudaDeviceSynchronize();
  printf("per step: remainder/smem %.0f  fast/smem %.0f  remainder/global %.0f  fast/global %.0f cycles\n",
         cyc[0] / 40.0, cyc[1] / 40.0, cyc[2] / 40.0, cyc[3] / 40.0);
}
