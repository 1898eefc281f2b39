// internal.hpp — kernel argument blocks and launcher declarations shared by the
// CUDA translation unit (kernels.cu) and the C++ host layer (capi.cpp).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace gpm {

// One kernel group of the exact GP (gp.hpp:81-92) as uploaded to the device.
struct GroupDev {
  const double* pts;   // FP64 SoA [(5 + n_out)][ns]: zs0..zs3, zn(+ln sv), alpha_0..alpha_{n_out-1}
  const double* ilt64; // FP64 L^{-T} [n][n] row-major (upper triangular, zeros below)
  const float* ilt32;  // FP32 copy of L^{-T}
  const float* zs32;   // FP32 scaled inputs [4][n]
  const float* tc_b;   // tensor-core operand: L^{-T} hi/lo TF32 tiles (see kernels_tc.cu)
  const int4* tc_meta; // per (pass, chunk): float offset, ncols, col0
  int tc_npad, tc_np, tc_npass;
  double ls[4];
  double sv, log_sv;
  int n_out;
  int out_idx[kMaxOutPerGroup];
};
struct ModelDev {
  int n, m, G;
  int ns;  // stride of the pts SoA arrays: n rounded up to even (padded points contribute 0)
  GroupDev g[kMaxGroups];
};

enum { NOISE_PHILOX = 0, NOISE_INJECTED = 1 };

struct RolloutArgs {
  ModelDev model;
  int model_kind;
  NominalDev nom;
  Edd5Dev edd5;
  int K_local;
  long long s_begin;
  int T;
  int n_obs;
  double lo[2], hi[2];
  double sv, sw;  // noise standard deviations
  int noise_mode;
  const double* eps;  // injected [K_local][T][2]
  uint64_t key;
  const double* nominal_seq;
  const double* tw;
  int R;
  const TaskDev* task;
  const double* r_bar;
  const double* margins;
  const double* x0;
  double* cost_mean;
  float4* queries;
  uint32_t* viol_bits;
  uint32_t* coll_bits;
  uint8_t* term;
  uint8_t* alive;
  int words;  // ceil(T/32)
  double* scratch;  // per lane-group trajectory scratch (rollout_scratch_doubles)
};

struct VarianceArgs {
  const float4* queries;  // [KT]
  long long KT;
  int n;
  GroupDev g;
  double coef;   // Σ over the group's outputs of w_terrain^2 (trace coefficient)
  int accumulate; // 0: trace = coef*var, 1: trace += coef*var
  double* trace; // [KT]
};

struct ReduceArgs {
  int K_local;
  long long s_begin;
  int T;
  double lambda;
  const double* cost_mean;
  const double* trace;  // may be null (no GP)
  double var_w;
  int noise_mode;
  const double* eps;
  uint64_t key;
  double sv, sw;
  double* costs_out;
  double* e_out;
  double* partials;
  unsigned int* ticket;
  double* rank_tuple;
  int finish;
  double* nominal_seq;
  double lo[2], hi[2];
  double* out;  // [2 + 6]: command, best, mean, ess, entropy, nonfinite, N
  long long K_total;
};

struct TightenArgs {
  ModelDev model;
  int model_kind;
  NominalDev nom;
  int T;
  const double* tw;
  int R;
  const double* x0;
  const double* nominal_seq;
  const TaskDev* task;
  double chi2, z;
  double* horizon_cov;
  double* r_bar;
  double* margins;
  int* infeasible;
  // scratch of the three-phase pass
  double* tq;         // [T][4] GP queries at the belief means
  double* tmu;        // [T+1][5] belief means
  double* tJ;         // [T][25] Jacobians
  double* tvar_part;  // [T][G][splits] partial ||L^{-1}k*||^2
};

// launchers (kernels.cu); all enqueue on `st` and return cudaGetLastError()
cudaError_t launch_rollout(const RolloutArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_variance(const VarianceArgs& a, int path, cudaStream_t st);
cudaError_t launch_reduce(const ReduceArgs& a, int blocks, cudaStream_t st);
cudaError_t launch_finish(const double* tuples, int n, int T, double lambda, double* nominal_seq,
                          const double lo[2], const double hi[2], double* out, long long K_total,
                          double* combined, cudaStream_t st);
cudaError_t launch_tighten(const TightenArgs& a, cudaStream_t st);
cudaError_t launch_predict(const ModelDev& m, const double* q, long long S, double* mean,
                           double* var, cudaStream_t st);
cudaError_t launch_philox_noise(uint64_t key, long long s_begin, int K, int T, double sv,
                                double sw, double* eps, cudaStream_t st);
size_t rollout_smem_bytes(const RolloutArgs& a);
size_t rollout_scratch_doubles(int T, int num_sms);
int reduce_blocks_for(int K_local, int num_sms);
int tighten_splits(int n);
void build_tc_operand(const double* ilt, int n, std::vector<float>& data, std::vector<int4>& meta,
                      int& n_pad, int& np, int& n_pass);
void tc_profile_read(double* out);
void count_launch(int n = 1);
unsigned long long launches_total();

}  // namespace gpm
