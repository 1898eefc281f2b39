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

// ---------------------------------------------------------------------------
// Hyperparameter grid (select_kernel_grid, gp.cpp:274-366) on the device: every grid
// cell (signal_var, shared scale, noise_var) is one CTA that builds its kernel matrix
// K = sv·exp(-d2 / 2s²) + nv·I from the shared scaled squared distances, factors it
// (blocked left-looking Cholesky, 32-column panels; failure = a pivot not > 0, as
// Eigen's LLT) and scores the summed log marginal likelihood
//   Σ_j -½ y_jᵀ K⁻¹ y_j - Σ log L_ii - ½ n log 2π,  y_jᵀ K⁻¹ y_j = ‖L⁻¹ y_j‖²
// (one forward solve per output). Load-time work, FP64 throughout; the cell order and
// the first-strictly-greater argmax stay on the host as in the reference.
namespace {

constexpr int GB = 32;   // panel width
constexpr int GK = 64;   // k-chunk of the panel update staged in shared memory

__global__ void __launch_bounds__(256, 1) lml_grid_kernel(const double* __restrict__ d2, const double* __restrict__ yc,
                                                          int n, int m, const double* __restrict__ cells,
                                                          double* __restrict__ work, double* __restrict__ score) {
  __shared__ double bt[GB][GK + 1];  // panel rows' k-chunk (the 32 pivot rows of block J)
  __shared__ double dblk[GB][GB + 1];
  __shared__ int fail;
  __shared__ double red[8];
  const int cell = blockIdx.x;
  const double sv = cells[3 * cell], s = cells[3 * cell + 1], nv = cells[3 * cell + 2];
  const double cexp = -1.0 / (2.0 * s * s);
  double* M = work + (size_t)cell * n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // K, lower triangle (gp.cpp:304-305): sv * exp(-d2 / (2 s^2)), + nv on the diagonal
  for (size_t idx = tid; idx < (size_t)n * n; idx += blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    if (j <= i) M[idx] = sv * exp(d2[idx] * cexp) + (i == j ? nv : 0.0);
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int j0 = 0; j0 < n; j0 += GB) {
    const int w = min(GB, n - j0);
    // (a) panel update: M[i][j0 + c] -= Σ_{k < j0} M[i][k] M[j0 + c][k], rows i >= j0
    //     lane = panel column c, warps stride the rows; pivot rows staged per k-chunk
    double acc[8];  // rows warp + 8 r of this pass
    for (int ib = j0; ib < n; ib += 64) {
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r] = 0.0;
      for (int k0 = 0; k0 < j0; k0 += GK) {
        const int kw = min(GK, j0 - k0);
        __syncthreads();
        for (int t = tid; t < GB * GK; t += blockDim.x) {
          const int c = t / GK, k = t % GK;
          bt[c][k] = (c < w && k < kw) ? M[(size_t)(j0 + c) * n + k0 + k] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int i = ib + warp + 8 * r;
          if (i < n) {
            const double* mi = M + (size_t)i * n + k0;
            double a = acc[r];
            for (int k = 0; k < kw; ++k) a = fma(mi[k], bt[lane][k], a);  // mi[k]: one broadcast load per warp
            acc[r] = a;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = ib + warp + 8 * r;
        if (i < n && lane < w && j0 + lane <= i) M[(size_t)i * n + j0 + lane] -= acc[r];
      }
    }
    __syncthreads();
    // (b) diagonal block: unblocked Cholesky by warp 0 (lane = row)
    for (int t = tid; t < GB * GB; t += blockDim.x) {
      const int r = t / GB, c = t % GB;
      dblk[r][c] = (r < w && c <= r) ? M[(size_t)(j0 + r) * n + j0 + c] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      for (int c = 0; c < w; ++c) {
        double p = dblk[c][c];
        for (int k = 0; k < c; ++k) p -= dblk[c][k] * dblk[c][k];
        if (!(p > 0.0)) {
          if (lane == 0) fail = 1;
          break;
        }
        const double d = sqrt(p);
        if (lane > c && lane < w) {
          double v = dblk[lane][c];
          for (int k = 0; k < c; ++k) v -= dblk[lane][k] * dblk[c][k];
          dblk[lane][c] = v / d;
        }
        __syncwarp();
        if (lane == 0) dblk[c][c] = d;
        __syncwarp();
      }
    }
    __syncthreads();
    if (fail) break;
    for (int t = tid; t < GB * GB; t += blockDim.x) {
      const int r = t / GB, c = t % GB;
      if (r < w && c <= r) M[(size_t)(j0 + r) * n + j0 + c] = dblk[r][c];
    }
    // (c) rows below the block: L[i][j0 + c] = (M[i][j0 + c] - Σ_{k<c} L[i][j0+k] D[c][k]) / D[c][c]
    for (int i = j0 + w + warp; i < n; i += 8) {
      double x = lane < w ? M[(size_t)i * n + j0 + lane] : 0.0;
      for (int c = 0; c < w; ++c) {
        const double xc = __shfl_sync(0xffffffffu, x / dblk[c][c], c);
        if (lane == c) x = xc;
        if (lane > c) x -= xc * dblk[lane][c];
      }
      if (lane < w) M[(size_t)i * n + j0 + lane] = x;
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) score[cell] = -INFINITY;
    return;
  }
  // logdet = Σ log L_ii (gp.cpp:307)
  double ld = 0.0;
  for (int i = tid; i < n; i += blockDim.x) ld += log(M[(size_t)i * n + i]);
  for (int o = 16; o; o >>= 1) ld += __shfl_xor_sync(0xffffffffu, ld, o);
  if (lane == 0) red[warp] = ld;
  __syncthreads();
  double logdet = 0.0;
  for (int q = 0; q < 8; ++q) logdet += red[q];
  __syncthreads();
  // forward solves, one warp per output: z = L^{-1} y_j, quad_j = ‖z‖² (written over y's slot)
  extern __shared__ double zbuf[];  // [8][n]
  double* z = zbuf + (size_t)warp * n;
  double quad_sum = 0.0;
  for (int j = warp; j < m; j += 8) {
    const double* y = yc + (size_t)j * n;
    double q = 0.0;
    for (int i = 0; i < n; ++i) {
      const double* li = M + (size_t)i * n;
      double sdot = 0.0;
      for (int k = lane; k < i; k += 32) sdot = fma(li[k], z[k], sdot);
      for (int o = 16; o; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
      const double zi = (y[i] - sdot) / li[i];
      if (lane == 0) z[i] = zi;
      q = fma(zi, zi, q);
      __syncwarp();
    }
    quad_sum += q;
  }
  if (lane == 0) red[warp] = quad_sum;
  __syncthreads();
  if (tid == 0) {
    double qs = 0.0;
    for (int q = 0; q < 8; ++q) qs += red[q];
    const double log2pi = log(2.0 * gpm::kPi);
    score[cell] = -0.5 * qs - (double)m * logdet - 0.5 * (double)m * (double)n * log2pi;
  }
}

}  // namespace

namespace gpm {

// Scores of the given cells ((sv, s, nv) triples) for scaled squared distances d2 (n x n,
// host) and outputs Y (n x m, row-major, host). -inf marks a failed factorisation.
cudaError_t device_lml_grid(const double* d2, const double* Y, int n, int m, const double* cells, int n_cells,
                            double* scores) {
  double *dd2 = nullptr, *dy = nullptr, *dc = nullptr, *dw = nullptr, *ds = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaSuccess;
  std::vector<double> yc((size_t)n * m);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) yc[(size_t)j * n + i] = Y[(size_t)i * m + j];
  const size_t smem = sizeof(double) * 8 * (size_t)n;
#define GRID_CK(call)                  \
  do {                                 \
    if ((e = (call)) != cudaSuccess) { \
      goto done;                       \
    }                                  \
  } while (0)
  GRID_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  GRID_CK(cudaMalloc(&dd2, sizeof(double) * (size_t)n * n));
  GRID_CK(cudaMalloc(&dy, sizeof(double) * yc.size()));
  GRID_CK(cudaMalloc(&dc, sizeof(double) * 3 * (size_t)n_cells));
  GRID_CK(cudaMalloc(&dw, sizeof(double) * (size_t)n * n * n_cells));
  GRID_CK(cudaMalloc(&ds, sizeof(double) * (size_t)n_cells));
  GRID_CK(cudaMemcpyAsync(dd2, d2, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice, st));
  GRID_CK(cudaMemcpyAsync(dy, yc.data(), sizeof(double) * yc.size(), cudaMemcpyHostToDevice, st));
  GRID_CK(cudaMemcpyAsync(dc, cells, sizeof(double) * 3 * (size_t)n_cells, cudaMemcpyHostToDevice, st));
  GRID_CK(cudaFuncSetAttribute(lml_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  lml_grid_kernel<<<n_cells, 256, smem, st>>>(dd2, dy, n, m, dc, dw, ds);
  count_launch();
  GRID_CK(cudaGetLastError());
  GRID_CK(cudaMemcpyAsync(scores, ds, sizeof(double) * (size_t)n_cells, cudaMemcpyDeviceToHost, st));
  GRID_CK(cudaStreamSynchronize(st));
#undef GRID_CK
done:
  cudaFree(dd2);
  cudaFree(dy);
  cudaFree(dc);
  cudaFree(dw);
  cudaFree(ds);
  if (st) cudaStreamDestroy(st);
  return e;
}

}  // namespace gpm
