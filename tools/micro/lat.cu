// Latency probes for the tightening mean chain's primitives (single warp / block):
// dependent DFMA, dependent FFMA, 64-bit SHFL, LDS.64, BAR.SYNC (4 warps), MUFU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[256];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = fmaf(f, (float)b, (float)a);
  long long t2 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = __shfl_xor_sync(0xffffffffu, y, 1) + 0.0;
  long long t3 = clock64();
  int idx = threadIdx.x & 7;
  double z = 0.0;
  for (int i = 0; i < n; ++i) {
    z = sm[idx];
    idx = ((int)z + i) & 7;
  }
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t5 = clock64();
  double w = y;
  for (int i = 0; i < n; ++i) w = w + b;
  long long t6 = clock64();
  double m = w;
  for (int i = 0; i < n; ++i) m = m * b;
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    cyc[5] = t6 - t5; cyc[6] = t7 - t6;
  }
  out[threadIdx.x] = x + f + y + z + w + m;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 256 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) probe<<<1, 128>>>(out, cyc, 0.5, 0.999, n);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA dep", "FFMA dep", "SHFL.64+DADD dep", "LDS.64 dep (+IADD/F2I)", "BAR.SYNC 4 warps", "DADD dep", "DMUL dep"};
  for (int i = 0; i < 7; ++i) printf("%-26s %.1f cyc\n", names[i], (double)cyc[i] / n);
  return 0;
}
