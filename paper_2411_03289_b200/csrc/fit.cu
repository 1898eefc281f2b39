// Device FP64 factorisation for GpModel::fit at large n.
//
// Replaces the host loops of factor_group for the O(n^3) part: the Cholesky of
// K + (noise_var + jitter) I with the jitter ladder (gp.cpp:116-133) and the
// triangular inverse L^{-1} (gp.cpp:135-138). Load-time work: at n = 2048 that is
// ~2.9 GFLOP for the factor and ~2.9 GFLOP for the inverse, seconds as scalar host
// loops. Everything stays in FP64; only the summation order differs from the host
// (warp-strided dot products), so factors agree to rounding.
//
// Layout: row-major n x n, L lower (zeros above), X = L^{-1} lower. Both fit in L2
// (32 MiB each at n = 2048), so the column/row sweeps below run out of L2.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "internal.hpp"

namespace {

// Left-looking column j: v_i = A_ij (+ diag_add if i == j) - sum_{k<j} L_ik L_jk for
// i in [j, n). One warp per row; lanes stride k, so row loads are coalesced and the
// pivot row L_j stays in L1 for every warp of the block.
__global__ void __launch_bounds__(256) chol_column_dots(const double* __restrict__ A,
                                                        const double* __restrict__ L,
                                                        double* __restrict__ v, int n, int j,
                                                        double diag_add) {
  const int lane = threadIdx.x & 31;
  const int i = j + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= n) return;
  const double* li = L + (size_t)i * n;
  const double* lj = L + (size_t)j * n;
  double s0 = 0.0, s1 = 0.0;
  int k = lane;
  for (; k + 32 < j; k += 64) {
    s0 = fma(li[k], lj[k], s0);
    s1 = fma(li[k + 32], lj[k + 32], s1);
  }
  if (k < j) s0 = fma(li[k], lj[k], s0);
  double s = s0 + s1;
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    double a = A[(size_t)i * n + j];
    if (i == j) a += diag_add;
    v[i] = a - s;
  }
}

// L_jj = sqrt(v_j), L_ij = v_i / L_jj. A pivot that is not > 0 (Eigen LLT's failure
// test, NaN included) raises the flag; the column is then left at zero.
__global__ void chol_column_scale(double* __restrict__ L, const double* __restrict__ v, int n,
                                  int j, int* __restrict__ fail) {
  const int i = j + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= n) return;
  const double p = v[j];
  if (!(p > 0.0)) {
    if (i == j) *fail = 1;
    return;
  }
  const double d = sqrt(p);
  L[(size_t)i * n + j] = i == j ? d : v[i] / d;
}

// Row i of X = L^{-1}: X_ic = (delta_ic - sum_{k=c}^{i-1} L_ik X_kc) / L_ii for c <= i.
// A block owns 32 consecutive columns (lane = column, coalesced 256-byte row segments
// of X); its 8 warps stride k and meet in shared memory. X_kc = 0 for k < c, so every
// lane runs the same k range.
__global__ void __launch_bounds__(256) lower_inverse_row(const double* __restrict__ L,
                                                         double* __restrict__ X, int n, int i) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 32;
  const int c = c0 + lane;
  const double* li = L + (size_t)i * n;
  double s0 = 0.0, s1 = 0.0;
  int k = c0 + warp;
  for (; k + 8 < i; k += 16) {
    s0 = fma(li[k], X[(size_t)k * n + c], s0);
    s1 = fma(li[k + 8], X[(size_t)(k + 8) * n + c], s1);
  }
  if (k < i) s0 = fma(li[k], X[(size_t)k * n + c], s0);
  part[warp][lane] = s0 + s1;
  __syncthreads();
  if (warp == 0 && c <= i) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += part[w][lane];
    X[(size_t)i * n + c] = ((c == i ? 1.0 : 0.0) - s) / li[i];
  }
}

}  // namespace

namespace gpm {

// K: n x n symmetric kernel matrix without the noise/jitter diagonal. Runs the jitter
// ladder {0, 1e-10, ..., 1e-6} on the device (gp.cpp:116-133); on success writes L and
// L^{-1} (row-major, lower) and the jitter used and sets *ok. Returns the first CUDA
// error (the caller turns it into GPMPPI_CUDA_ERROR).
cudaError_t device_factor(const double* K, int n, double noise_var, double* L_out, double* X_out,
                          double* jitter_out, bool* ok) {
  const size_t bytes = (size_t)n * n * sizeof(double);
  double *dA = nullptr, *dL = nullptr, *dv = nullptr;
  int* dfail = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaSuccess;
  *ok = false;
#define FIT_CK(call)                   \
  do {                                 \
    if ((e = (call)) != cudaSuccess) { \
      goto done;                       \
    }                                  \
  } while (0)
  FIT_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  FIT_CK(cudaMalloc(&dA, bytes));
  FIT_CK(cudaMalloc(&dL, bytes));
  FIT_CK(cudaMalloc(&dv, (size_t)n * sizeof(double)));
  FIT_CK(cudaMalloc(&dfail, sizeof(int)));
  FIT_CK(cudaMemcpyAsync(dA, K, bytes, cudaMemcpyHostToDevice, st));
  for (int attempt = 0; attempt <= 5 && !*ok; ++attempt) {
    const double jitter = attempt == 0 ? 0.0 : std::pow(10.0, -11 + attempt);
    int fail = 1;
    FIT_CK(cudaMemsetAsync(dL, 0, bytes, st));
    FIT_CK(cudaMemsetAsync(dfail, 0, sizeof(int), st));
    for (int j = 0; j < n; ++j) {
      const int rows = n - j;
      chol_column_dots<<<(rows + 7) / 8, 256, 0, st>>>(dA, dL, dv, n, j, noise_var + jitter);
      chol_column_scale<<<(rows + 255) / 256, 256, 0, st>>>(dL, dv, n, j, dfail);
    }
    count_launch(2 * n);
    FIT_CK(cudaGetLastError());
    FIT_CK(cudaMemcpyAsync(&fail, dfail, sizeof(int), cudaMemcpyDeviceToHost, st));
    FIT_CK(cudaStreamSynchronize(st));
    if (!fail) {
      *ok = true;
      *jitter_out = jitter;
    }
  }
  if (*ok) {
    double* dX = dA;  // K is no longer needed
    FIT_CK(cudaMemsetAsync(dX, 0, bytes, st));
    for (int i = 0; i < n; ++i) lower_inverse_row<<<i / 32 + 1, 256, 0, st>>>(dL, dX, n, i);
    count_launch(n);
    FIT_CK(cudaGetLastError());
    FIT_CK(cudaMemcpyAsync(L_out, dL, bytes, cudaMemcpyDeviceToHost, st));
    FIT_CK(cudaMemcpyAsync(X_out, dX, bytes, cudaMemcpyDeviceToHost, st));
    FIT_CK(cudaStreamSynchronize(st));
  }
#undef FIT_CK
done:
  cudaFree(dA);
  cudaFree(dL);
  cudaFree(dv);
  cudaFree(dfail);
  if (st) cudaStreamDestroy(st);
  return e;
}

}  // namespace gpm
