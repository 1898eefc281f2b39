// internal.hpp — kernel argument blocks and launcher declarations shared by the
// CUDA translation unit (kernels.cu) and the C++ host layer (capi.cpp).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <vector>

#include "common.cuh"

namespace gpm {

// One kernel group of the exact GP (gp.hpp:81-92) as uploaded to the device.
struct GroupDev {
  const double* pts;   // FP64 SoA [(5 + n_out)][ns]: zs0..zs3, zn(+ln sv), alpha_0..alpha_{n_out-1}
  const double* ilt64; // FP64 L^{-T} [n][n] row-major (upper triangular, zeros below)
  const double* linv64; // FP64 L^{-1} [n][n] row-major (lower): row j = column j of L^{-T}
  const float* ilt32;  // FP32 copy of L^{-T}
  const float* zs32;   // FP32 scaled inputs [4][n]
  const float* tc_b;   // tensor-core operand: L^{-T} hi/lo TF32 tiles (see kernels_tc.cu)
  const int4* tc_meta; // per (pass, chunk): float offset, ncols, col0
  int tc_npad, tc_np, tc_npass;
  const uint16_t* tc_h;  // 3xFP16 operand: scaled L^{-T} hi/lo FP16 blocks (build_tc_operand_f16)
  const int4* tc_hmeta;  // per (pass, chunk): fp16 offset, ncols, col0
  double tc_hfac;        // (sf2 / operand scale)^2
  const uint16_t* tc_h2;   // CTA-pair 3xFP16 operand (build_tc_operand_f16x2): per (512-column pass,
  const int4* tc_h2meta;   // chunk) one record [CTA0 part | CTA1 part]; meta .x offset, .w part size
  int tc_npass2;           // 512-column passes
  double ls[4];
  double sv, log_sv;
  int n_out;
  int out_idx[kMaxOutPerGroup];
};
struct ModelDev {
  int n, m, G;
  int ns;  // stride of the pts SoA arrays: n rounded up to even (padded points contribute 0)
  // 1 when every real point's exponent row zn (= -|z|^2/2 + ln sv) lies in [-600, 600] and
  // |ln sv| <= 50: the rollout then folds exp(zn_j) into its combined alpha rows and forms
  // the kernel-row exponent without zn (q·z + qn <= |z|^2/2 stays far from FP64 overflow)
  int fold_zn;
  GroupDev g[kMaxGroups];
};

enum { NOISE_PHILOX = 0, NOISE_INJECTED = 1 };

// Per-robot strides of the batched planner state (B independent planners that
// share one GP model; B = 1 is the single Planner). Robot b's slice of an array
// with stride S starts at b*S.
struct BatchStrides {
  // per-robot tick block: x0[0..4], [5] variance weight of the task, [6] Philox key
  // (bit pattern), [7] the tick's sequence number (zero-copy completion words) -- one H2D
  // copy stages everything a robot's tick needs
  static constexpr int X0 = 8;
  // terrain weights [kMaxTerrains], then the per-group variance coefficients
  // Σ_o w(o)² over each kernel group's outputs [kMaxGroups] (mppi.cpp:34-49; host-computed)
  static constexpr int TW = kMaxTerrains + kMaxGroups;
  static constexpr int TW_COEF = kMaxTerrains;
  static constexpr int OUT = 16;                  // command + diagnostics
  GPM_HD static int nom(int T) { return 2 * T; }
  GPM_HD static int rbar(int T) { return T; }
  GPM_HD static int marg(int T) { return T * kMaxObstacles; }  // [T][n_obs] inside
};

// GPM_COOP=1 compiles the co-resident variance experiment's query-progress publication into
// the rollout (an A/B build: python -m paper_2411_03289_b200.build --variant=coop -DGPM_COOP=1,
// then GPMPPI_LIB=.../libgpmppi_b200_coop.so GPMPPI_COOP=1); the default build leaves it out.
#ifndef GPM_COOP
#define GPM_COOP 0
#endif

// Lane-group geometry of the GP rollout, fixed per planner (rollout_geometry): LPS lanes
// per sample group, SPG samples per group, `threads` per block, spb samples per work item
// (one block's chunk of one robot), chunks = items per robot.
struct RolloutGeom {
  int lps, spg, threads, spb, chunks;
};
// Query / variance-trace slot of (robot-major sample slot sl, step k): item-major, so the
// block working on an item writes its step-k queries contiguously ([item][k][spb]) and the
// variance tiles of early steps are complete while the chains are still running.
GPM_HD long long query_slot(long long sl, int k, int K_local, int T, int spb, int chunks) {
  const long long b = sl / K_local;
  const int ls = (int)(sl - b * K_local);
  const long long item = b * chunks + ls / spb;
  return (item * T + k) * spb + ls % spb;
}

struct RolloutArgs {
  ModelDev model;
  int model_kind;
  NominalDev nom;
  Edd5Dev edd5;
  int B;              // robots
  int K_local;        // samples per robot on this device
  long long K_total;  // samples per robot in the whole (possibly sharded) solve
  long long s_begin;
  int T;
  int n_obs_max;      // max obstacles over the robots (shared-memory sizing)
  double lo[2], hi[2];
  double sv, sw;  // noise standard deviations
  int noise_mode;
  const double* eps;  // injected [B][K_local][T][2]
  double* noise_out;  // Philox mode: the drawn noise, same layout (the reduce reads it back)
  const double* nominal_seq;  // [B][2T]
  const double* tw;           // [B][kMaxTerrains]
  int R;
  const TaskDev* task;        // [B]
  const double* r_bar;        // [B][T]
  const double* margins;      // [B][T*kMaxObstacles]
  const double* x0;           // [B][8]
  double* cost_mean;          // [B*K_local]
  float4* queries;            // [B*K_local*T]
  uint32_t* viol_bits;        // [B*K_local*words]
  uint32_t* coll_bits;
  uint8_t* term;
  uint8_t* alive;
  int words;  // ceil(T/32)
  double* scratch;  // per lane-group trajectory scratch (rollout_scratch_doubles)
  int scratch_smem;  // set by launch_rollout: the trajectory scratch fits in shared memory (after ubuf)
  RolloutGeom geom;  // rollout_geometry of the planner (query layout, query_slot)
  int smem_budget;   // dynamic shared memory cap of the rollout block (0: 227 KB)
  unsigned long long* progress;  // [items * groups per block]: steps whose queries a group has
                                 // written (release), read by the concurrent variance kernel; null: off
};

struct VarianceArgs {
  const float4* queries;  // [KT]
  long long KT;
  int n;
  GroupDev g;
  double coef;    // multiplier of var (1 in the solve: the reduce applies Σ w² per robot)
  int accumulate; // 0: out = coef*var, 1: out += coef*var
  double* trace;  // [KT] (this group's slice)
};

struct ReduceArgs {
  RolloutGeom geom;  // the trace is in query_slot order
  unsigned long long* progress;  // rollout query-progress words to re-arm (null: none)
  long long progress_words;
  int B;
  int K_local;
  long long K_total;
  long long s_begin;
  int T;
  int bpr;  // blocks per robot
  double lambda;
  const double* cost_mean;  // [B*K_local]
  const double* var;        // [G][B*K_local*T] raw per-group variances (null: no GP)
  int G;
  const double* tw;         // [B][TW] terrain weights + per-group trace coefficients (BatchStrides::TW_COEF)
  const double* x0;         // [B][8] robot tick blocks (variance weight, key)
  int noise_mode;
  const double* eps;
  double sv, sw;
  double* costs_out;
  double* e_out;
  double* partials;       // [B*bpr][W]
  unsigned int* ticket;   // [B]
  double* rank_tuple;     // [B][W]
  int finish;
  double* nominal_seq;    // [B][2T]
  double lo[2], hi[2];
  double* out;            // [B][16]: command, best, mean, ess, entropy, nonfinite, N
  double* out_host;       // null, or mapped pinned [B][16]: the same + the tick's sequence in [15]
};

struct TightenArgs {
  ModelDev model;
  int model_kind;
  NominalDev nom;
  int B;
  int T;
  const double* tw;  // [B][kMaxTerrains]
  int R;
  const double* x0;           // [B][8]
  const double* nominal_seq;  // [B][2T]
  const TaskDev* task;        // [B]
  double chi2, z;
  double* horizon_cov;  // [B][25T]
  double* r_bar;        // [B][T]
  double* margins;      // [B][T*kMaxObstacles]
  int* infeasible;      // [B]
  double* done_host;    // null, or mapped pinned [B][2]: infeasible, tick sequence (x0 block [7])
  // scratch of the three-phase pass
  double* tq;         // [B][T][4] GP queries at the belief means
  double* tmu;        // [B][T+1][5] belief means
  double* tJ;         // [B][T][25] Jacobians
  double* tvar_part;  // [B][T][G][splits] partial ||L^{-1}k*||^2
  // single-robot pipelining: the mean kernel's publisher warp counts the steps whose GP query
  // (flag 0) and Jacobian / belief mean (flag 1) are out; the variance block of step k starts
  // at query k and counts step k's finished slices (flags[2 + k]); the covariance kernel runs
  // the recursion and thresholds step by step behind them and lowers every flag at its end.
  // Null: grid ordering only (batched planners).
  unsigned int* tflags;  // [T + 2]: queries out, J / belief means out, per-step variance slices done
  double* tcv;           // [T][2] combined correction variances of the pipelined pass
  double* cmd_host;      // non-null: the mean kernel publishes the command (cmd_dev, OUT words) here
  const double* cmd_dev;
};

// Programmatic dependent launch: the kernel may be scheduled while its stream
// predecessor finishes; it must execute pdl_wait() (griddepcontrol.wait) before it
// reads anything the predecessor wrote. Predecessors call pdl_trigger() once all their
// CTAs are resident (single-wave kernels: at entry).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const int no_pdl = getenv("GPMPPI_NO_PDL") ? atoi(getenv("GPMPPI_NO_PDL")) : 0;  // diagnostics
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#if defined(__CUDACC__)
// release / acquire at GPU scope: the rollout publishes how many steps of queries a lane
// group has written; the concurrent variance kernel acquires before reading them
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// tick timeline (diagnostics, -DGPM_TIMELINE): %globaltimer at fixed points, slot i keeps the
// latest (even i) or the earliest (odd i) stamp of the tick
#ifdef GPM_TIMELINE
static __device__ unsigned long long g_tl[32];  // one per translation unit (timeline_read merges them)
__device__ __forceinline__ void tl_stamp(int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (i & 1)
    atomicMin(&g_tl[i], t);
  else
    atomicMax(&g_tl[i], t);
}
#else
__device__ __forceinline__ void tl_stamp(int) {}
#endif
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
#endif

// launchers (kernels.cu); all enqueue on `st` and return cudaGetLastError()
// copies the tick's staged inputs (mapped pinned memory) into device memory: the tick graph's
// first node (a copy-engine node costs ~9 us more between the launch and the first kernel)
cudaError_t launch_stage_tick(const void* src_mapped, void* dst, size_t bytes, cudaStream_t st);
cudaError_t launch_rollout(const RolloutArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_variance(const VarianceArgs& a, int path, cudaStream_t st);
cudaError_t launch_reduce(const ReduceArgs& a, int blocks, cudaStream_t st);
cudaError_t launch_finish(const double* tuples, int n, int T, double lambda, double* nominal_seq,
                          const double lo[2], const double hi[2], double* out, long long K_total,
                          double* combined, cudaStream_t st, double* out_host = nullptr,
                          const double* x0_block = nullptr);
// max_warps: warps per rollout block (8; 7 leaves the registers of a co-resident variance block)
RolloutGeom rollout_geometry(int K_local, int B, int T, int n_pts, int G, int num_sms, int max_warps = 8);
size_t rollout_launch_smem(const RolloutArgs& a, int* scratch_smem);
// kernels_tc.cu: the co-resident variance (variance_coop_kernel) and its shared memory
size_t coop_smem_bytes(const GroupDev& g, int stages);
cudaError_t launch_variance_coop(const VarianceArgs& v, const unsigned long long* progress, long long progress_words,
                                 int T, const RolloutGeom& geom, size_t rollout_smem, int num_sms, cudaStream_t st);
// slots of the item-major query / trace arrays (>= B*K_local*T: the last chunk of a robot is padded)
GPM_HD long long query_slots(const RolloutGeom& g, int B, int T) { return (long long)B * g.chunks * T * g.spb; }
cudaError_t launch_tighten(const TightenArgs& a, cudaStream_t st);
cudaError_t launch_predict(const ModelDev& m, const double* q, long long S, double* mean,
                           double* var, cudaStream_t st);
// reference free functions (mppi.hpp:60-79)
cudaError_t launch_rollout_one(const ModelDev& M, int model_kind, const NominalDev& nom, const Edd5Dev& edd,
                               const double* x0, const double* seq, int T, const double* w, int R,
                               double* states, double* corr, cudaStream_t st);
cudaError_t launch_trajectory_weights(const double* c, long long K, double lambda, double* w, cudaStream_t st);
cudaError_t launch_update_controls(const double* nom, int T, const double* eps, const double* w, long long K,
                                   const double lo[2], const double hi[2], double* out, cudaStream_t st);
cudaError_t launch_shift_horizon(const double* seq, int T, double* out, cudaStream_t st);
cudaError_t launch_philox_noise(uint64_t key, long long s_begin, int K, int T, double sv,
                                double sw, double* eps, cudaStream_t st);
size_t rollout_smem_bytes(const RolloutArgs& a);
size_t rollout_scratch_doubles(int T, int num_sms);
int reduce_blocks_for(int K_local, int B, int num_sms, int T);
int tighten_splits(int n, int B);
// CTA-pair variance (variance_f16x2_kernel): the MMAs of 512-column pass p, 16-point chunk kb.
// The chunk's active columns (triangle skip at GPM_PAIR_GRAN granularity, widths rounded to 32
// so each CTA's N/2 rows stay whole 8-row groups) form one contiguous range of pass-relative
// TMEM columns; it is issued as at most two M = 256 MMAs: c0[s] = first TMEM column, nc[s] =
// N (0 = no MMA), split at the 256-column boundary. GPM_PAIR_BALANCE=1 splits a range wider
// than 256 columns into two near-equal MMAs instead (the microbenchmark's max(75, N/2)-cycle
// pair MMA favours it), but measured slower: config 2 variance 0.132 -> 0.139 ms, config 3
// 7.73 -> 7.95 ms. Shared by the kernel and the host operand builder, which must agree.
#ifndef GPM_PAIR_GRAN
#define GPM_PAIR_GRAN 32  // column granularity of the triangle skip (a compile-time power of two)
#endif
#ifndef GPM_PAIR_BALANCE
#define GPM_PAIR_BALANCE 0
#endif
GPM_HD void pair2_cols(int p, int kb, int n_pad, int* c0, int* nc) {
  const int npw = n_pad - 512 * p < 512 ? n_pad - 512 * p : 512;
  const int rel = 16 * kb - 512 * p;
  int lo = -1, hi = 0;  // active range [lo, hi) of pass-relative TMEM columns
  for (int h = 0; h < 2; ++h) {
    int w = npw - 256 * h;
    w = w < 0 ? 0 : (w > 256 ? 256 : w);
    const int r = rel - 256 * h;
    const int c = r <= 0 ? 0 : (r & ~(GPM_PAIR_GRAN - 1));
    const int wr = (w + 31) & ~31;
    c0[h] = 256 * h + c;
    nc[h] = (w > 0 && c < w) ? wr - c : 0;
    if (nc[h] > 0) {
      if (lo < 0) lo = c0[h];
      hi = c0[h] + nc[h];
    }
  }
#if GPM_PAIR_BALANCE
  if (nc[0] > 0 && nc[1] > 0) {  // contiguous: half 0 then runs to column 256 (w = 256 there)
    const int total = hi - lo;
    const int na = ((total >> 1) + 31) & ~31;
    c0[0] = lo;
    nc[0] = na;
    c0[1] = lo + na;
    nc[1] = total - na;
  }
#endif
}
void build_tc_operand_f16x2(const double* ilt, int n, double sv, int n_pad, std::vector<uint16_t>& data,
                            std::vector<int4>& meta, int& n_pass2);
void build_tc_operand_f16(const double* ilt, int n, double sv, int n_pad, int np, int n_pass,
                          std::vector<uint16_t>& data, std::vector<int4>& meta, double& hfac);
void build_tc_operand(const double* ilt, int n, std::vector<float>& data, std::vector<int4>& meta,
                      int& n_pad, int& np, int& n_pass);
void tc_profile_read(double* out);
void tc_trace_read(double* out);  // 64 clock64 stamps of CTA 0 (GPMPPI_TC_DEBUG bit 4096)
void timeline_read(double* out);  // 32 %globaltimer stamps of the last tick (-DGPM_TIMELINE builds), read-and-reset
void timeline_read_unit(unsigned long long* h);  // kernels_tc.cu's copy of the stamps, read-and-reset
void count_launch(int n = 1);
// fit.cu: device Cholesky (jitter ladder) + L^{-1} for GpModel::fit at large n.
cudaError_t device_factor(const double* K, int n, double noise_var, double* L_out, double* X_out,
                          double* jitter_out, bool* ok);
unsigned long long launches_total();
// fit.cu: summed LML of each hyperparameter grid cell (sv, s, nv) on the device (-inf: LLT failed)
cudaError_t device_lml_grid(const double* d2, const double* Y, int n, int m, const double* cells, int n_cells,
                            double* scores);

}  // namespace gpm
