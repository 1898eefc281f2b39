// kernels.cu — sm_100a kernels of the GP-MPPI solve (mppi.cpp:389-462).
//
//   rollout_gp_kernel     one warp per sample: Philox/injected noise, clamp,
//                         FP64 GP-mean (k*·alpha, gp.cpp:172-182) + dynamic
//                         unicycle (dynamics.cpp:39-66) + per-step costs and
//                         flags (costs.cpp:127-171); writes the step queries.
//   rollout_base_kernel   one thread per sample for the GP-free models.
//   variance_ffma_kernel  flash-style var = sf2 - ||k* L^{-T}||^2 (gp.cpp:184-191)
//                         with k* recomputed on the fly, FP32 FFMA, FP64 sum.
//   reduce_kernel         costs, min-baselined softmax, Σw·eps, ESS/entropy
//                         as one tuple per block; the last block combines the
//                         tuples, updates/clamps/shifts (mppi.cpp:125-173).
//   tighten_kernel        tightening pass (mppi.cpp:250-282), FP64.
//   predict_kernel        GpModel::predict_batch in FP64 (gp.cpp:152-198).
#include <cuda_runtime.h>

#include <atomic>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "internal.hpp"

namespace gpm {

static std::atomic<unsigned long long> g_launches{0};
void count_launch(int n) { g_launches += n; }
unsigned long long launches_total() { return g_launches.load(); }

// -------------------------------------------------------------------------
// warp helpers (xor butterfly: every lane ends with bit-identical sums)
GPM_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
GPM_D double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// -------------------------------------------------------------------------
// 2^(j/32), j < 32: the exp_tab table (common.cuh), staged into shared memory per block
__constant__ double kExp2Frac[32] = {
    0x1.0000000000000p+0, 0x1.059b0d3158574p+0, 0x1.0b5586cf9890fp+0, 0x1.11301d0125b51p+0,
    0x1.172b83c7d517bp+0, 0x1.1d4873168b9aap+0, 0x1.2387a6e756238p+0, 0x1.29e9df51fdee1p+0,
    0x1.306fe0a31b715p+0, 0x1.371a7373aa9cbp+0, 0x1.3dea64c123422p+0, 0x1.44e086061892dp+0,
    0x1.4bfdad5362a27p+0, 0x1.5342b569d4f82p+0, 0x1.5ab07dd485429p+0, 0x1.6247eb03a5585p+0,
    0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, 0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0,
    0x1.8ace5422aa0dbp+0, 0x1.93737b0cdc5e5p+0, 0x1.9c49182a3f090p+0, 0x1.a5503b23e255dp+0,
    0x1.ae89f995ad3adp+0, 0x1.b7f76f2fb5e47p+0, 0x1.c199bdd85529cp+0, 0x1.cb720dcef9069p+0,
    0x1.d5818dcfba487p+0, 0x1.dfc97337b9b5fp+0, 0x1.ea4afa2a490dap+0, 0x1.f50765b6e4540p+0};

// -------------------------------------------------------------------------
// Rollout, GP ensemble model (terrain-combined alpha: two sums per kernel group whatever the
// output count). LPS lanes per sample group, SPG samples per group (compile time).
size_t rollout_smem_bytes(const RolloutArgs& a) {
  size_t b = sizeof(TaskDev);
  b += sizeof(double) * (size_t)(2 * a.T + a.T + a.T * (a.n_obs_max > 0 ? a.n_obs_max : 1) + a.R + 2 + 32);
  b = (b + 15) & ~(size_t)15;
  if (a.model_kind == MODEL_GP)
    b += sizeof(double) * (size_t)7 * a.model.ns * a.model.G;  // per group: Z (5 rows) + combined alpha (2 rows)
  return b;
}

struct SmemView {
  TaskDev* task;
  double* nom;
  double* rbar;
  double* marg;
  double* tw;
  double* etab;  // 2^(j/32), j < 32
  double* pts;   // groups back to back
};

GPM_D SmemView carve_smem(const RolloutArgs& a, unsigned char* smem) {
  SmemView v;
  v.task = reinterpret_cast<TaskDev*>(smem);
  double* p = reinterpret_cast<double*>(smem + sizeof(TaskDev));
  v.nom = p;
  p += 2 * a.T;
  v.rbar = p;
  p += a.T;
  v.marg = p;
  p += a.T * (a.n_obs_max > 0 ? a.n_obs_max : 1);
  v.tw = p;
  p += a.R + 2;
  v.etab = p;
  p += 32;
  // 16-byte align by pointer arithmetic on the shared array (an integer round trip
  // would turn every access into a generic LD instead of LDS)
  size_t off = (size_t)(reinterpret_cast<unsigned char*>(p) - smem);
  off = (off + 15) & ~(size_t)15;
  v.pts = reinterpret_cast<double*>(smem + off);
  for (int i = threadIdx.x; i < 32; i += blockDim.x) v.etab[i] = kExp2Frac[i];
  return v;
}

// Robot b's per-tick view (task, nominal sequence, thresholds, terrain weights).
GPM_D void load_robot_smem(const RolloutArgs& a, const SmemView& v, int b) {
  const int nw = sizeof(TaskDev) / 8;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.task + b);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(v.task);
  for (int i = threadIdx.x; i < nw; i += blockDim.x) dst[i] = src[i];
  const double* nom = a.nominal_seq + (size_t)b * BatchStrides::nom(a.T);
  for (int i = threadIdx.x; i < 2 * a.T; i += blockDim.x) v.nom[i] = nom[i];
  const double* rb = a.r_bar + (size_t)b * BatchStrides::rbar(a.T);
  for (int i = threadIdx.x; i < a.T; i += blockDim.x) v.rbar[i] = rb[i];
  const double* mg = a.margins + (size_t)b * BatchStrides::marg(a.T);
  for (int i = threadIdx.x; i < a.T * a.n_obs_max; i += blockDim.x) v.marg[i] = mg[i];
  const double* tw = a.tw + (size_t)b * BatchStrides::TW;
  for (int i = threadIdx.x; i < a.R; i += blockDim.x) v.tw[i] = tw[i];
  if (a.model_kind == MODEL_GP) {
    // combine_terrains (mppi.cpp:34-49) is linear in the per-output GP means, so it is
    // folded into alpha once per robot and tick: alpha~_v = Σ_o w(o) alpha_o over the
    // v-channel outputs (ascending o), likewise omega. The serial chain then carries 2
    // sums per group instead of n_out (2 FMAs and 2 loads per point-sample, not n_out).
    double* gp = v.pts;
    const int ns = a.model.ns;
    for (int g = 0; g < a.model.G; ++g) {
      const GroupDev& G = a.model.g[g];
      for (int j = threadIdx.x; j < ns; j += blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        for (int o0 = 0; o0 < G.n_out; o0 += kOutChunk) {  // ascending o, kOutChunk loads in flight
          double al[kOutChunk];
#pragma unroll
          for (int o = 0; o < kOutChunk; ++o)
            al[o] = o0 + o < G.n_out ? __ldg(G.pts + (size_t)(5 + o0 + o) * ns + j) : 0.0;
#pragma unroll
          for (int o = 0; o < kOutChunk; ++o) {
            if (o0 + o < G.n_out) {
              const int gi = G.out_idx[o0 + o];
              if (gi & 1)
                s1 = fma(tw[gi >> 1], al[o], s1);
              else
                s0 = fma(tw[gi >> 1], al[o], s0);
            }
          }
        }
        if (a.model.fold_zn) {  // exp(zn_j) folded into the combined rows (ModelDev::fold_zn)
          const double ez = exp(__ldg(G.pts + (size_t)4 * ns + j));
          s0 *= ez;
          s1 *= ez;
        }
        gp[5 * ns + j] = s0;
        gp[6 * ns + j] = s1;
      }
      gp += 7 * ns;
    }
  }
}

// sl = robot-major local sample index (b*K_local + local s); s = global counter index
GPM_D void sample_noise(const RolloutArgs& a, uint64_t key, long long sl, long long s, int k, double* e0,
                        double* e1) {
  if (a.noise_mode == NOISE_INJECTED) {
    const double2 e = reinterpret_cast<const double2*>(a.eps)[(size_t)sl * a.T + k];
    *e0 = e.x;
    *e1 = e.y;
  } else {
    double z1, z2;
    philox_gaussian_pair(key, (uint64_t)s, (uint32_t)k, &z1, &z2);
    *e0 = a.sv * z1;
    *e1 = a.sw * z2;
  }
}

template <int LPS>
GPM_D double group_sum(double v) {  // xor butterfly inside an LPS-lane group
#pragma unroll
  for (int o = LPS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sums NV (<= LPS) values across an LPS-lane group and returns every total in every
// lane: a transpose reduction (LPS-1 shuffles: each level halves the values a lane
// carries) leaves total i in lane i of the group, then NV broadcasts. A butterfly
// per value costs NV*log2(LPS) shuffles.
template <int LPS, int NV>
GPM_D void group_allsum(double (&val)[NV]) {
  static_assert(NV <= LPS, "group_allsum: at most one value per lane");
  const int gl = threadIdx.x & (LPS - 1);
  double t[LPS];
#pragma unroll
  for (int i = 0; i < LPS; ++i) t[i] = i < NV ? val[i] : 0.0;
#pragma unroll
  for (int lvl = LPS / 2; lvl >= 1; lvl >>= 1) {
    const bool up = gl & lvl;
#pragma unroll
    for (int i = 0; i < lvl; ++i) {
      const double send = up ? t[i] : t[i + lvl];
      t[i] = (up ? t[i + lvl] : t[i]) + __shfl_xor_sync(0xffffffffu, send, lvl);
    }
  }
  const int base = (threadIdx.x & 31) & ~(LPS - 1);
#pragma unroll
  for (int i = 0; i < NV; ++i) val[i] = __shfl_sync(0xffffffffu, t[0], base + i);
}

// One LPS-lane group per SPG samples (32/LPS groups per warp share every Z/alpha
// shared-memory read; each lane reuses its loaded points for its group's SPG samples,
// which halves the LDS per FP64 op at SPG=2 and gives SPG independent exp chains).
// The GP query of step k needs only (v_k, omega_k, u_k), so:
//  phase 1 (serial in k): noise, clamp, GP mean k*·alpha (lanes split the n
//          points, butterfly sum), first-order lag update of (v, omega);
//  phase 2 (lanes split the steps k, one sample after the other): heading recursion,
//          FP64 sincos / exact-arc increments, x/y in step order, non-finite freeze
//          (mppi.cpp:343-346), per-step costs and flags (costs.cpp:127-171).
// Per-sample trajectory scratch lives in L2 (scr, 9 arrays of T+1 doubles).
constexpr int SCR_ARRAYS = 9;
#ifndef GPM_ROLL_UNROLL
#define GPM_ROLL_UNROLL 16
#endif
constexpr int kRollUnroll = GPM_ROLL_UNROLL;  // point pairs in flight per lane and sample in the GP loop
constexpr int kMaxSampleSlotsPerBlock = 128;  // groups per block x SPG: <= 64 x 2, 8 x 4
#ifndef GPM_ROLLOUT_MINB
#define GPM_ROLLOUT_MINB 1
#endif
// Phase 2 of one sample (lanes split the steps): heading recursion, FP64 sincos /
// exact-arc increments, x/y in step order, non-finite freeze (mppi.cpp:343-346),
// per-step costs and flags (costs.cpp:127-171); scr holds the sample's phase-1 chain.
template <int LPS>
GPM_D void rollout_phase2(const RolloutArgs& a, const SmemView& sv, const TaskDev& task, double* scr,
                          const double* x0, int T, int stride, int gl, bool valid, long long sl, int O) {
  double* su0 = scr;
  double* su1 = scr + stride;
  double* sv_ = scr + 2 * stride;
  double* sw = scr + 3 * stride;
  double* sth = scr + 4 * stride;
  double* ssin = scr + 5 * stride;
  double* scos = scr + 6 * stride;
  double* sx = scr + 7 * stride;
  double* sy = scr + 8 * stride;
  (void)su1;
#ifdef GPM_ROLLOUT_TRACE
  const bool trc = blockIdx.x == 0 && threadIdx.x == 0;
  long long p2t[5];
  p2t[0] = clock64();
#endif
  // ---------------- phase 2a: heading recursion (arc_advance: theta = wrap(theta + omega dt))
  if (gl == 0) {  // omega read 8 steps ahead of the chain (one load latency per 8 steps)
    double th = x0[2];
    sth[0] = th;
    for (int k0 = 0; k0 < T; k0 += 8) {
      double wv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) wv[i] = k0 + i < T ? sw[k0 + i] : 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (k0 + i < T) {
          th = th + wv[i] * a.nom.dt;
          if (!(th > -kPi && th <= kPi)) th = wrap_angle_fast(th);  // remainder is the identity on (-π, π]
          sth[k0 + i + 1] = th;
        }
    }
  }
  __syncwarp();
#ifdef GPM_ROLLOUT_TRACE
  p2t[1] = clock64();
#endif
  // ---------------- phase 2b: sincos and exact-arc increments, lanes split the steps
  for (int k = gl; k < T; k += LPS) {
    const double th = sth[k], vk = sv_[k], wk = sw[k];
    double sp, cp;
    sincos(th, &sp, &cp);
    ssin[k] = sp;
    scos[k] = cp;
    double dx = 0.0, dy = 0.0, t2 = th;
    arc_advance(dx, dy, t2, vk, 0.0, wk, a.nom.dt, sp, cp);
    sx[k + 1] = dx;
    sy[k + 1] = dy;
  }
  __syncwarp();
#ifdef GPM_ROLLOUT_TRACE
  p2t[2] = clock64();
#endif
  // ---------------- phase 2c: positions in step order + first non-finite state
  int kd = T;  // states k > kd are frozen at state kd (mppi.cpp:343-346)
  if (gl == 0) {  // increments of 8 steps loaded ahead of the prefix sum (step order)
    double x = x0[0], y = x0[1];
    sx[0] = x;
    sy[0] = y;
    for (int k0 = 0; k0 < T; k0 += 8) {
      double dxv[8], dyv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = k0 + i < T ? k0 + i : T - 1;
        dxv[i] = sx[k + 1];
        dyv[i] = sy[k + 1];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (k0 + i < T) {
          x += dxv[i];
          y += dyv[i];
          sx[k0 + i + 1] = x;
          sy[k0 + i + 1] = y;
        }
    }
  }
  __syncwarp();
  // first non-finite state (mppi.cpp:343-346): lanes check their steps, group minimum
  for (int k = gl; k < T; k += LPS)
    if (!(isfinite(sx[k + 1]) && isfinite(sy[k + 1]) && isfinite(sth[k + 1]) && isfinite(sv_[k + 1]) &&
          isfinite(sw[k + 1]))) {
      kd = k;
      break;
    }
#pragma unroll
  for (int o = LPS / 2; o > 0; o >>= 1) kd = min(kd, __shfl_xor_sync(0xffffffffu, kd, o));
  __syncwarp();
#ifdef GPM_ROLLOUT_TRACE
  p2t[3] = clock64();
#endif
  // ---------------- phase 2d: per-step costs and flags (costs.cpp:127-171), lanes split the steps
  double cost = 0.0;
  double decay = 1.0;  // 0.9^k by repeated multiplication, as costs.cpp:146 (continued across
  int kdec = 0;        // this lane's increasing steps: the same product sequence, fewer multiplies)
  for (int wd = 0; wd < a.words; ++wd) {
    uint32_t vb = 0, cb = 0;
    const int kend = min(T, 32 * wd + 32);
    for (int k = 32 * wd + gl; k < kend; k += LPS) {
      const int ip = min(k, kd), in = min(k + 1, kd);
      const double prev[5] = {sx[ip], sy[ip], sth[ip], sv_[ip], sw[ip]};
      const double next[5] = {sx[in], sy[in], sth[in], sv_[in], sw[in]};
      for (; kdec < k; ++kdec) decay *= 0.9;
      const StepCost c = step_cost(task, prev, next, ssin[ip], scos[ip], sv.rbar[k],
                                   sv.marg + (size_t)k * O, su0[k], decay);
      cost += c.cost;
      vb |= (uint32_t)c.viol << (k & 31);
      cb |= (uint32_t)c.coll << (k & 31);
    }
#pragma unroll
    for (int o = LPS / 2; o > 0; o >>= 1) {
      vb |= __shfl_xor_sync(0xffffffffu, vb, o);
      cb |= __shfl_xor_sync(0xffffffffu, cb, o);
    }
    if (valid && gl == 0) {
      a.viol_bits[(size_t)sl * a.words + wd] = vb;
      a.coll_bits[(size_t)sl * a.words + wd] = cb;
    }
  }
  cost = group_sum<LPS>(cost);
  const bool alive = valid && kd == T;
  bool term = false;
  if (task.kind == TASK_AVOIDANCE) {  // costs.cpp:169 terminal_cost
    const int il = min(T, kd);
    const double gx = sx[il] - task.goal[0], gy = sy[il] - task.goal[1];
    term = sqrt(gx * gx + gy * gy) <= task.goal[2];
    cost += task.aw[3] * (term ? 0.0 : task.high_cost);
  }
  if (valid && gl == 0) {
    a.cost_mean[sl] = alive ? cost : __longlong_as_double(0x7ff8000000000000LL);
    a.term[sl] = term;
    a.alive[sl] = alive;
  }
#ifdef GPM_ROLLOUT_TRACE
  if (trc) {
    p2t[4] = clock64();
    printf("phase2: heading %lld arcs %lld positions %lld costs %lld\n", p2t[1] - p2t[0], p2t[2] - p2t[1],
           p2t[3] - p2t[2], p2t[4] - p2t[3]);
  }
#endif
}

#ifndef GPM_EXP_PRESCALE
#define GPM_EXP_PRESCALE 1
#endif
#ifndef GPM_QUERY_BULK
#define GPM_QUERY_BULK 1
#endif
template <int LPS, int SPG, bool FOLD>
__global__ void __launch_bounds__(256, GPM_ROLLOUT_MINB) rollout_gp_kernel(const RolloutArgs a) {
  if (threadIdx.x == 0) tl_stamp(1);
  pdl_trigger();  // single wave: the variance grid may be scheduled (it waits for this grid)
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemView sv = carve_smem(a, smem);
  const int ns = a.model.ns;  // even SoA stride (padding points contribute exactly 0)
  const int T = a.T;
  const int gl = threadIdx.x % LPS;  // lane inside the sample group
  const int groups_per_block = blockDim.x / LPS;
  const int gib = threadIdx.x / LPS;  // group index in the block
  double2* ubuf;  // this group's clamped controls u[SPG][T], drawn before the serial chain
  double* scr_sm;  // shared-memory trajectory scratch (a.scratch_smem), after every ubuf
  {  // stage Z / alpha of every group (SoA) into shared memory, once per block
    double* dst = sv.pts;
    for (int g = 0; g < a.model.G; ++g) {
      const int cnt = 5 * ns;  // Z rows; the combined alpha rows are per robot (load_robot_smem)
      const double2* src = reinterpret_cast<const double2*>(a.model.g[g].pts);
      double2* d2 = reinterpret_cast<double2*>(dst);
#pragma unroll 4
      for (int i = threadIdx.x; i < cnt / 2; i += blockDim.x) {
        double2 z = __ldg(src + i);
#if GPM_EXP_PRESCALE  // the exponent rows carry exp_tab_t's 32/ln2 (padding: -1e300·46 stays finite)
        z.x *= kInvLn2x32;
        z.y *= kInvLn2x32;
#endif
        d2[i] = z;
      }
      dst += 7 * ns;
    }
    ubuf = reinterpret_cast<double2*>(dst) + (size_t)gib * SPG * T;
    scr_sm = reinterpret_cast<double*>(reinterpret_cast<double2*>(dst) + (size_t)groups_per_block * SPG * T);
  }
  __shared__ double gil[kMaxGroups][4];  // reciprocal lengthscales: no FP64 divide on the chain
  if (threadIdx.x < 4 * a.model.G) gil[threadIdx.x >> 2][threadIdx.x & 3] = 1.0 / a.model.g[threadIdx.x >> 2].ls[threadIdx.x & 3];
  pdl_wait();  // model staging above overlapped the predecessor; per-tick inputs below
  const TaskDev& task = *sv.task;
  const int stride = T + 1;
  // scratch slot of sample j of this group
  // (shared memory when the launcher found room: the phase-2 serial loops then wait on
  // LDS latency instead of L2 round trips)
  double* const scr0 = a.scratch_smem ? scr_sm + (size_t)gib * SPG * SCR_ARRAYS * stride
                                      : a.scratch + ((size_t)blockIdx.x * kMaxSampleSlotsPerBlock + (size_t)gib * SPG) *
                                                        SCR_ARRAYS * stride;
  const double av = a.nom.dt / a.nom.tau_v, aw = a.nom.dt / a.nom.tau_omega;
  // work items: (robot, chunk of groups_per_block*SPG samples); every lane of the block
  // runs the same item sequence (samples beyond K are masked, never early-exit)
  const int spb = groups_per_block * SPG;  // == a.geom.spb
  const int chunks = a.geom.chunks;
  const long long items = (long long)a.B * chunks;
  int loaded = -1;

  for (long long item = blockIdx.x; item < items; item += gridDim.x) {
#ifdef GPM_ROLLOUT_TRACE
    const long long t_item = clock64();
#endif
    const int b = (int)(item / chunks);
    const int ls0 = (int)(item % chunks) * spb + gib * SPG;  // first local sample of the group
    if (b != loaded) {
      __syncthreads();  // previous item's readers are done with the robot view
      load_robot_smem(a, sv, b);
      __syncthreads();
      loaded = b;
    }
    const double* x0 = a.x0 + (size_t)b * BatchStrides::X0;
    const uint64_t key = (uint64_t)__double_as_longlong(x0[6]);
    const int O = task.n_obs;
    bool valid[SPG];
    long long sl[SPG], s[SPG];
    double v[SPG], w[SPG];
#pragma unroll
    for (int j = 0; j < SPG; ++j) {
      const int ls = ls0 + j;
      valid[j] = ls < a.K_local;
      sl[j] = (long long)b * a.K_local + (valid[j] ? ls : 0);  // output slot
      s[j] = a.s_begin + (valid[j] ? ls : 0);                  // noise counter (per-robot key)
      v[j] = x0[3];
      w[j] = x0[4];
      if (gl == 0) {
        double* scr = scr0 + (size_t)j * SCR_ARRAYS * stride;
        scr[2 * stride] = v[j];
        scr[3 * stride] = w[j];
      }
    }
    // noise + clamp of every (sample, step) up front, lanes split the pairs: the draws
    // do not depend on the chain, so they leave the serial path (mppi.cpp:298-308)
    for (int idx0 = gl; idx0 < SPG * T; idx0 += 2 * LPS) {  // two draws per lane in flight (ILP)
      double e0[2], e1[2];
      int jj[2], kk[2];
      bool vjs[2], in[2];
      long long slj[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = idx0 + u * LPS;
        in[u] = idx < SPG * T;
        const int j = (SPG == 1 || !in[u]) ? 0 : idx / T;
        kk[u] = SPG == 1 ? idx : (in[u] ? idx % T : 0);
        jj[u] = j;
        bool vj = valid[0];
        long long sj = sl[0], cj = s[0];
#pragma unroll
        for (int q = 1; q < SPG; ++q) {
          vj = j == q ? valid[q] : vj;
          sj = j == q ? sl[q] : sj;
          cj = j == q ? s[q] : cj;
        }
        vjs[u] = in[u] && vj;
        slj[u] = sj;
        e0[u] = e1[u] = 0.0;
        if (vjs[u]) sample_noise(a, key, sj, cj, kk[u], &e0[u], &e1[u]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!in[u]) continue;
        const int j = jj[u], k = kk[u];
        if (vjs[u] && a.noise_out)
          reinterpret_cast<double2*>(a.noise_out)[(size_t)slj[u] * T + k] = make_double2(e0[u], e1[u]);
        const double u0 = clampd(sv.nom[2 * k] + e0[u], a.lo[0], a.hi[0]);
        const double u1 = clampd(sv.nom[2 * k + 1] + e1[u], a.lo[1], a.hi[1]);
        ubuf[j * T + k] = make_double2(u0, u1);
        if (vjs[u]) {
          double* scr = scr0 + (size_t)j * SCR_ARRAYS * stride;
          scr[k] = u0;
          scr[stride + k] = u1;
        }
      }
    }
    __syncwarp();
#ifdef GPM_ROLLOUT_TRACE
    const long long t_p1 = clock64();
#endif
    // ---------------- phase 1: serial (v, omega) chains with the GP mean
    for (int k = 0; k < T; ++k) {
      double u0[SPG], u1[SPG];
#pragma unroll
      for (int j = 0; j < SPG; ++j) {
        const double2 u = ubuf[j * T + k];
        u0[j] = u.x;
        u1[j] = u.y;
#if GPM_COOP || !GPM_QUERY_BULK
        if (valid[j] && gl == 0)  // item-major slot: (item, k, sample within the item)
          a.queries[(size_t)((item * T + k) * spb + ls0 + j - (item % chunks) * spb)] =
              make_float4((float)v[j], (float)w[j], (float)u0[j], (float)u1[j]);
#endif
      }
#if GPM_COOP
      if (a.progress && gl == 0)  // steps < k+1 of this group's queries are published
        st_release_u64(a.progress + (size_t)item * groups_per_block + gib, (unsigned long long)(k + 1));
#endif
      double cm0[SPG], cm1[SPG];  // combine_terrains (mppi.cpp:34-49)
#pragma unroll
      for (int j = 0; j < SPG; ++j) cm0[j] = cm1[j] = 0.0;
      const double* gp = sv.pts;
      for (int g = 0; g < a.model.G; ++g) {
        // gp.cpp:172-176 augmented query [q/l | -1/2|q/l|^2 | 1]
        double q0[SPG], q1[SPG], q2[SPG], q3[SPG], qn[SPG];
        double acc[SPG][2];  // terrain-combined v / omega means (load_robot_smem)
#pragma unroll
        for (int j = 0; j < SPG; ++j) {
          q0[j] = v[j] * gil[g][0];  // q/l (gp.cpp:172-176) by reciprocal: <= 1 ulp from the division
          q1[j] = w[j] * gil[g][1];
          q2[j] = u0[j] * gil[g][2];
          q3[j] = u1[j] * gil[g][3];
          qn[j] = -0.5 * (q0[j] * q0[j] + q1[j] * q1[j] + q2[j] * q2[j] + q3[j] * q3[j]);
#if GPM_EXP_PRESCALE
          qn[j] *= kInvLn2x32;
#endif
          acc[j][0] = acc[j][1] = 0.0;
        }
        // two adjacent points per lane and load (LDS.128): the 32/LPS sample groups of a
        // warp read the same addresses, so a 16-byte access doubles the bytes per wavefront
        const double2* z0 = reinterpret_cast<const double2*>(gp);
        const double2* z1 = reinterpret_cast<const double2*>(gp + ns);
        const double2* z2 = reinterpret_cast<const double2*>(gp + 2 * ns);
        const double2* z3 = reinterpret_cast<const double2*>(gp + 3 * ns);
        const double2* zn = reinterpret_cast<const double2*>(gp + 4 * ns);
        const double2* cv = reinterpret_cast<const double2*>(gp + 5 * ns);
        const double2* cw = reinterpret_cast<const double2*>(gp + 6 * ns);
        const int half = ns >> 1;
#pragma unroll(kRollUnroll / SPG)
        for (int jp = gl; jp < half; jp += LPS) {
          // gp.cpp:177-179: k*_j = exp(q_aug · inputs_aug_j)
          const double2 a0 = z0[jp], a1 = z1[jp], a2 = z2[jp], a3 = z3[jp];
          const double2 an = FOLD ? make_double2(0.0, 0.0) : zn[jp];
          const double2 av = cv[jp], aw = cw[jp];
#pragma unroll
          for (int j = 0; j < SPG; ++j) {
            // q·z + (qn + zn) as one DADD and four DFMAs (gp.cpp:177-179); with FOLD the zn
            // factor rides in the alpha rows and the exponent is q·z + qn (four DFMAs, one
            // load fewer per point pair)
            const double e0 = FOLD ? qn[j] : qn[j] + an.x, e1 = FOLD ? qn[j] : qn[j] + an.y;
            const double d0 = fma(q0[j], a0.x, fma(q1[j], a1.x, fma(q2[j], a2.x, fma(q3[j], a3.x, e0))));
            const double d1 = fma(q0[j], a0.y, fma(q1[j], a1.y, fma(q2[j], a2.y, fma(q3[j], a3.y, e1))));
#if GPM_EXP_PRESCALE  // d = 32/ln2 · (q·z + qn + zn): the reduction is one DADD (exp_tab_t)
            const double k0 = exp_tab_t(d0, sv.etab), k1 = exp_tab_t(d1, sv.etab);
#else
            const double k0 = exp_tab(d0, sv.etab), k1 = exp_tab(d1, sv.etab);
#endif
            acc[j][0] = fma(k1, av.y, fma(k0, av.x, acc[j][0]));  // gp.cpp:181-182, terrain-combined
            acc[j][1] = fma(k1, aw.y, fma(k0, aw.x, acc[j][1]));
          }
        }
        if constexpr (SPG * 2 <= LPS) {  // all group sums at once (transpose reduction)
          double tot[SPG * 2];
#pragma unroll
          for (int j = 0; j < SPG; ++j) {
            tot[2 * j] = acc[j][0];
            tot[2 * j + 1] = acc[j][1];
          }
          group_allsum<LPS, SPG * 2>(tot);
#pragma unroll
          for (int j = 0; j < SPG; ++j) {
            cm0[j] += tot[2 * j];
            cm1[j] += tot[2 * j + 1];
          }
        } else {
#pragma unroll
          for (int j = 0; j < SPG; ++j) {
            cm0[j] += group_sum<LPS>(acc[j][0]);
            cm1[j] += group_sum<LPS>(acc[j][1]);
          }
        }
        gp += (size_t)7 * ns;
      }
#pragma unroll
      for (int j = 0; j < SPG; ++j) {
        v[j] = v[j] + av * (u0[j] - v[j]) + cm0[j];  // step_nominal lag (dynamics.cpp:63-64) + mppi.cpp:341-342
        w[j] = w[j] + aw * (u1[j] - w[j]) + cm1[j];
        if (gl == 0) {
          double* scr = scr0 + (size_t)j * SCR_ARRAYS * stride;
          scr[2 * stride + k + 1] = v[j];
          scr[3 * stride + k + 1] = w[j];
        }
      }
    }
    __syncwarp();
#if !GPM_COOP && GPM_QUERY_BULK
    // the variance queries of every step, written after the chain from its state record (the
    // same doubles the chain used): the conversions and stores leave the serial path, and the
    // group's lanes split the (sample, step) pairs. Item-major slot: (item, k, sample in item).
    for (int idx = gl; idx < SPG * T; idx += LPS) {
      const int j = SPG == 1 ? 0 : idx / T, k = SPG == 1 ? idx : idx - j * T;
      bool vj = valid[0];
#pragma unroll
      for (int q = 1; q < SPG; ++q) vj = j == q ? valid[q] : vj;
      if (vj) {
        const double* scr = scr0 + (size_t)j * SCR_ARRAYS * stride;
        const double2 u = ubuf[j * T + k];
        a.queries[(size_t)((item * T + k) * spb + ls0 + j - (item % chunks) * spb)] =
            make_float4((float)scr[2 * stride + k], (float)scr[3 * stride + k], (float)u.x, (float)u.y);
      }
    }
#endif
#ifdef GPM_ROLLOUT_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0)
      printf("rollout item %lld: prologue %lld phase1 %lld (per step %lld)\n", item, t_p1 - t_item, clock64() - t_p1,
             (clock64() - t_p1) / T);
#endif
    if constexpr (SPG > 1 && LPS / SPG >= 2) {
      // phase 2 of the group's SPG samples side by side, LPS/SPG lanes each: their serial
      // heading / position recursions run in the same instructions instead of in turn
      constexpr int SUB = LPS / SPG;
      const int h = gl / SUB;
      bool vh = valid[0];
      long long slh = sl[0];
#pragma unroll
      for (int j = 1; j < SPG; ++j) {
        vh = h == j ? valid[j] : vh;
        slh = h == j ? sl[j] : slh;
      }
      rollout_phase2<SUB>(a, sv, task, scr0 + (size_t)h * SCR_ARRAYS * stride, x0, T, stride, gl % SUB, vh, slh, O);
      __syncwarp();
    } else {
      for (int j = 0; j < SPG; ++j) {  // phase 2, one sample after the other
        rollout_phase2<LPS>(a, sv, task, scr0 + (size_t)j * SCR_ARRAYS * stride, x0, T, stride, gl, valid[j], sl[j], O);
        __syncwarp();
      }
    }
  }
  if (threadIdx.x == 0) tl_stamp(0);
}

// GP-free models (mppi.cpp:351-368): one thread per sample; block = one robot chunk.
constexpr int kBaseSteps = 40;  // steps of controls drawn ahead of the GP-free chain (80 KB at 128 threads)
__global__ void __launch_bounds__(128) rollout_base_kernel(const RolloutArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemView sv = carve_smem(a, smem);
  const TaskDev& task = *sv.task;
  const int T = a.T;
  const int chunks = (a.K_local + blockDim.x - 1) / blockDim.x;
  const long long items = (long long)a.B * chunks;
  int loaded = -1;
  for (long long item = blockIdx.x; item < items; item += gridDim.x) {
    const int b = (int)(item / chunks);
    const int ls = (int)(item % chunks) * blockDim.x + threadIdx.x;
    if (b != loaded) {
      __syncthreads();
      load_robot_smem(a, sv, b);
      __syncthreads();
      loaded = b;
    }
    if (ls >= a.K_local) continue;
    const long long sl = (long long)b * a.K_local + ls;
    const long long s = a.s_begin + ls;
    const double* x0 = a.x0 + (size_t)b * BatchStrides::X0;
    const uint64_t key = (uint64_t)__double_as_longlong(x0[6]);
    const int O = task.n_obs;
    double st[5];
    for (int i = 0; i < 5; ++i) st[i] = x0[i];
    bool alive = true;
    double cost = 0.0, decay = 1.0;
    uint32_t vb = 0, cb = 0;
    // the noise and clamped controls of a chunk of kBaseSteps steps first (mppi.cpp:298-308):
    // they do not depend on the state chain, so the draws of consecutive steps overlap
    // instead of sitting on its serial path; [k][thread] in shared memory after the robot view
    double2* ub = reinterpret_cast<double2*>(sv.pts);
    for (int k = 0; k < T; ++k) {
      if (k % kBaseSteps == 0) {
        const int k1 = min(T, k + kBaseSteps);
        for (int kk = k; kk < k1; ++kk) {
          double e0, e1;
          sample_noise(a, key, sl, s, kk, &e0, &e1);
          if (a.noise_out) reinterpret_cast<double2*>(a.noise_out)[(size_t)sl * T + kk] = make_double2(e0, e1);
          ub[(size_t)(kk - k) * blockDim.x + threadIdx.x] = make_double2(
              clampd(sv.nom[2 * kk] + e0, a.lo[0], a.hi[0]), clampd(sv.nom[2 * kk + 1] + e1, a.lo[1], a.hi[1]));
        }
      }
      const double2 uk = ub[(size_t)(k % kBaseSteps) * blockDim.x + threadIdx.x];
      const double u[2] = {uk.x, uk.y};
      double sp, cp;  // heading of the step's start state: the dynamics and the cost share it
      sincos(st[2], &sp, &cp);
      double nx[5];
      if (alive) {
        if (a.model_kind == MODEL_EDD5) {
          step_edd5(st, u, a.edd5, a.nom.dt, nx);
        } else if (a.model_kind == MODEL_UNICYCLE) {
          step_kinematic(st, u, a.nom.dt, nx);
        } else {
          step_nominal(st, u, a.nom, nx, sp, cp);
        }
        if (!finite5(nx)) {
          alive = false;
          for (int i = 0; i < 5; ++i) nx[i] = st[i];
        }
      } else {
        for (int i = 0; i < 5; ++i) nx[i] = st[i];
      }
      const StepCost c = step_cost(task, st, nx, sp, cp, sv.rbar[k], sv.marg + (size_t)k * O, u[0], decay);
      cost += c.cost;
      decay *= 0.9;
      vb |= (uint32_t)c.viol << (k & 31);
      cb |= (uint32_t)c.coll << (k & 31);
      if ((k & 31) == 31 || k == T - 1) {
        a.viol_bits[(size_t)sl * a.words + (k >> 5)] = vb;
        a.coll_bits[(size_t)sl * a.words + (k >> 5)] = cb;
        vb = cb = 0;
      }
      for (int i = 0; i < 5; ++i) st[i] = nx[i];
    }
    bool term = false;
    if (task.kind == TASK_AVOIDANCE) {
      const double gx = st[0] - task.goal[0], gy = st[1] - task.goal[1];
      term = sqrt(gx * gx + gy * gy) <= task.goal[2];
      cost += task.aw[3] * (term ? 0.0 : task.high_cost);
    }
    a.cost_mean[sl] = alive ? cost : __longlong_as_double(0x7ff8000000000000LL);
    a.term[sl] = term;
    a.alive[sl] = alive;
  }
}

// lanes per sample group and samples per group (env GPMPPI_LPS / GPMPPI_SPG force them)
static int env_int(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}
// Lane-group layout of the GP rollout: LPS lanes per group, SPG samples per group.
// Measured on B200 (rollout ms): config2 (28 samples/SM) (8,1) 0.309, (16,2) 0.280,
// (8,2) 0.342; config5 (443/SM) (8,2) 3.31, (16,2) 3.70, (8,1) 4.54; config3 (16,2) 5.14,
// (8,1) 6.99. The 8-lane layout reads every Z/alpha byte four times per warp (LDS.128
// costs four wavefronts regardless of duplicate addresses) and is shared-memory bound;
// SPG = 2 halves the loads per FP64 op. GPMPPI_LPS / GPMPPI_SPG force a layout.
void rollout_layout(long long total, int num_sms, int* lps, int* spg) {
  static const int f_lps = env_int("GPMPPI_LPS"), f_spg = env_int("GPMPPI_SPG");
  const long long per_sm = (total + num_sms - 1) / num_sms;
  int l = per_sm >= 64 ? 8 : per_sm >= 7 ? 16 : 32;
  int g = 2;
  if (f_lps == 4 || f_lps == 8 || f_lps == 16 || f_lps == 32) l = f_lps;
  if (f_spg == 1 || f_spg == 2) g = f_spg;
  if (f_spg == 4) g = l == 32 ? 4 : 2;
  if (l == 4) g = 1;
  *lps = l;
  *spg = g;
}

// trajectory scratch for every sample slot the launcher can create
size_t rollout_scratch_doubles(int T, int num_sms) {
  return (size_t)GPM_ROLLOUT_MINB * num_sms * kMaxSampleSlotsPerBlock * SCR_ARRAYS * (size_t)(T + 1);
}

// Geometry of the GP rollout: spread all robots' samples over every SM in a single wave
// when possible (one block per SM); wider lane groups when n*T leaves no room for the
// control buffers (the shared-memory estimate assumes the maximum obstacle count, so the
// geometry -- and with it the query layout -- is fixed for the planner's lifetime).
RolloutGeom rollout_geometry(int K_local, int B, int T, int n_pts, int G, int num_sms, int max_warps) {
  const long long total = (long long)K_local * B;
  int lps = 8, spg = 1;
  rollout_layout(total, num_sms, &lps, &spg);
  auto shape = [&](int* threads, int* spb) {
    const int spw = 32 / lps * spg;
    const long long warps = (total + spw - 1) / spw;  // all robots' samples share the wave
    int wpb = (int)((warps + num_sms - 1) / num_sms);
    wpb = wpb < 1 ? 1 : (wpb > max_warps ? max_warps : wpb);
    *threads = wpb * 32;
    *spb = wpb * spw;
  };
  int threads = 32, spb = 1;
  shape(&threads, &spb);
  size_t base = sizeof(TaskDev) + sizeof(double) * (size_t)(2 * T + T + T * kMaxObstacles + kMaxTerrains + 2 + 32);
  base = ((base + 15) & ~(size_t)15) + sizeof(double) * (size_t)7 * ((n_pts + 1) & ~1) * (G > 0 ? G : 1);
  while (base + sizeof(double2) * (size_t)(threads / lps) * spg * T > 227 * 1024 && lps < 32) {
    lps *= 2;  // large n*T: wider groups, fewer control buffers
    shape(&threads, &spb);
  }
  RolloutGeom g;
  g.lps = lps;
  g.spg = spg;
  g.threads = threads;
  g.spb = spb;
  g.chunks = (K_local + spb - 1) / spb;
  return g;
}

// Dynamic shared memory of the GP rollout block: robot view + Z/alpha + control buffers,
// plus the trajectory scratch when it fits under a.smem_budget (bytes; 0 = the 227 KB
// per-block maximum -- the co-resident variance lowers it to leave room for its ring).
size_t rollout_launch_smem(const RolloutArgs& a, int* scratch_smem) {
  static int scr_env = -1;  // GPMPPI_SCR_GLOBAL=1 keeps the trajectory scratch in global memory
  if (scr_env < 0) {
    const char* e = getenv("GPMPPI_SCR_GLOBAL");
    scr_env = e ? atoi(e) : 0;
  }
  const size_t budget = a.smem_budget > 0 ? (size_t)a.smem_budget : 227 * 1024;
  const int lps = a.geom.lps, threads = a.geom.threads, spg = a.geom.spg;
  size_t smem_u = rollout_smem_bytes(a) + sizeof(double2) * (size_t)(threads / lps) * spg * a.T;
  const size_t scr_bytes = sizeof(double) * (size_t)(threads / lps) * spg * SCR_ARRAYS * (a.T + 1);
  const int in_smem = (!scr_env && smem_u + scr_bytes <= budget) ? 1 : 0;
  if (scratch_smem) *scratch_smem = in_smem;
  return smem_u + (in_smem ? scr_bytes : 0);
}

__global__ void __launch_bounds__(256) stage_tick_kernel(const ulonglong2* __restrict__ src, ulonglong2* dst, int n16,
                                                         const unsigned long long* __restrict__ src8,
                                                         unsigned long long* dst8, int n8) {
  if (threadIdx.x == 0) tl_stamp(17);
  pdl_trigger();  // the rollout's model staging may start; it waits for this grid's writes
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < n16; i += nt) dst[i] = src[i];  // PCIe reads of the mapped block
  for (int i = 2 * n16 + tid; i < n8; i += nt) dst8[i] = src8[i];
  if (threadIdx.x == 0) tl_stamp(16);
}

void timeline_read(double* out) {
#ifdef GPM_TIMELINE
  unsigned long long h[32], u[32];
  cudaMemcpyFromSymbol(h, g_tl, sizeof h);
  timeline_read_unit(u);
  for (int i = 0; i < 32; ++i) {
    const bool hv = (i & 1) ? h[i] != ~0ull && h[i] != 0ull : h[i] != 0ull;
    const bool uv = (i & 1) ? u[i] != ~0ull && u[i] != 0ull : u[i] != 0ull;
    const unsigned long long m = !hv ? u[i] : !uv ? h[i] : ((i & 1) ? (h[i] < u[i] ? h[i] : u[i]) : (h[i] > u[i] ? h[i] : u[i]));
    out[i] = (hv || uv) ? (double)m : 0.0;
  }
  for (int i = 0; i < 32; ++i) h[i] = (i & 1) ? ~0ull : 0ull;
  cudaMemcpyToSymbol(g_tl, h, sizeof h);
#else
  for (int i = 0; i < 32; ++i) out[i] = 0.0;
#endif
}

cudaError_t launch_stage_tick(const void* src_mapped, void* dst, size_t bytes, cudaStream_t st) {
  const int n8 = (int)(bytes / 8), n16 = n8 / 2;
  const int blocks = n16 / 256 < 1 ? 1 : (n16 / 256 > 148 ? 148 : n16 / 256);  // one 16-byte read per thread per round trip
  stage_tick_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const ulonglong2*>(src_mapped),
                                       reinterpret_cast<ulonglong2*>(dst), n16,
                                       reinterpret_cast<const unsigned long long*>(src_mapped),
                                       reinterpret_cast<unsigned long long*>(dst), n8);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_rollout(const RolloutArgs& a, int num_sms, cudaStream_t st) {
  const size_t smem = rollout_smem_bytes(a);
  if (a.K_local <= 0 || a.B <= 0) return cudaSuccess;
  if (a.model_kind == MODEL_GP) {
    const int lps = a.geom.lps, threads = a.geom.threads, spg = a.geom.spg;
    const long long items = (long long)a.B * a.geom.chunks;
    // one block per SM: capping registers for a second resident block (122 instead of
    // ~200) costs more ILP than the extra warps recover (config2 0.34 -> 0.52 ms)
    const long long cap = (long long)GPM_ROLLOUT_MINB * num_sms;
    const long long blocks = items < cap ? items : cap;
    using KF = void (*)(const RolloutArgs);
    // [fold zn][spg 1/2][lps]
    KF table[2][2][4] = {
        {{rollout_gp_kernel<4, 1, false>, rollout_gp_kernel<8, 1, false>, rollout_gp_kernel<16, 1, false>,
          rollout_gp_kernel<32, 1, false>},
         {rollout_gp_kernel<4, 1, false>, rollout_gp_kernel<8, 2, false>, rollout_gp_kernel<16, 2, false>,
          rollout_gp_kernel<32, 2, false>}},
        {{rollout_gp_kernel<4, 1, true>, rollout_gp_kernel<8, 1, true>, rollout_gp_kernel<16, 1, true>,
          rollout_gp_kernel<32, 1, true>},
         {rollout_gp_kernel<4, 1, true>, rollout_gp_kernel<8, 2, true>, rollout_gp_kernel<16, 2, true>,
          rollout_gp_kernel<32, 2, true>}}};
    const int li = lps == 4 ? 0 : lps == 8 ? 1 : lps == 16 ? 2 : 3;
    const int fz = a.model.fold_zn ? 1 : 0;
    // spg 4: one 32-lane group per warp carrying four samples (no duplicate addresses inside
    // a warp's Z/alpha loads, a quarter of the LDS instructions of the 8-lane layout)
    KF kern = spg == 4 ? (fz ? rollout_gp_kernel<32, 4, true> : rollout_gp_kernel<32, 4, false>)
                       : table[fz][spg == 2 ? 1 : 0][li];
    RolloutArgs ra = a;
    const size_t smem_u = rollout_launch_smem(a, &ra.scratch_smem);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_u);
    if (e != cudaSuccess) return e;
    e = launch_pdl(kern, dim3((unsigned)blocks), dim3(threads), smem_u, st, ra);
    if (e != cudaSuccess) return e;
  } else {
    const int threads = 128;
    const long long items = (long long)a.B * ((a.K_local + threads - 1) / threads);
    const long long blocks = items < (long long)num_sms * 8 ? items : (long long)num_sms * 8;
    const size_t smem_b = smem + sizeof(double2) * (size_t)threads * kBaseSteps;  // + the controls chunk
    cudaError_t e = cudaFuncSetAttribute(rollout_base_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
    if (e != cudaSuccess) return e;
    rollout_base_kernel<<<(unsigned)blocks, threads, smem_b, st>>>(a);
  }
  count_launch();
  return cudaGetLastError();
}

// -------------------------------------------------------------------------
// Variance (FP32 FFMA): per 64-query tile, column blocks of 128, row chunks of
// 32. k* recomputed per (column block, row chunk) in the exact-difference form
// exp(ln sf2 - 1/2 |q/l - z/l|^2) (no augmented-form cancellation in FP32).
constexpr int VQ = 64, VJ = 128, VI = 32;

__global__ void __launch_bounds__(256) variance_ffma_kernel(const VarianceArgs a) {
  __shared__ float qs[VQ][4];
  __shared__ __align__(16) float kT[VI][VQ];
  __shared__ __align__(16) float Ls[VI][VJ];
  const int n = a.n;
  const long long q0 = (long long)blockIdx.x * VQ;
  const int t = threadIdx.x, lane = t & 31, ty = t >> 5;
  if (t < VQ) {
    const long long qi = q0 + t;
    float4 q = qi < a.KT ? a.queries[qi] : make_float4(0.f, 0.f, 0.f, 0.f);
    qs[t][0] = q.x / (float)a.g.ls[0];
    qs[t][1] = q.y / (float)a.g.ls[1];
    qs[t][2] = q.z / (float)a.g.ls[2];
    qs[t][3] = q.w / (float)a.g.ls[3];
  }
  const float lsv = (float)a.g.log_sv;
  double part[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) part[i] = 0.0;
  for (int j0 = 0; j0 < n; j0 += VJ) {
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int d = 0; d < 4; ++d) acc[i][d] = 0.f;
    const int iend = min(n, j0 + VJ);
    for (int i0 = 0; i0 < iend; i0 += VI) {
      __syncthreads();
      // k* chunk: VI points × VQ queries (8 per thread)
      for (int e = t; e < VI * VQ; e += 256) {
        const int ii = e / VQ, qq = e % VQ;
        const int gi = i0 + ii;
        float v = 0.f;
        if (gi < n) {
          const float d0 = qs[qq][0] - a.g.zs32[gi];
          const float d1 = qs[qq][1] - a.g.zs32[n + gi];
          const float d2 = qs[qq][2] - a.g.zs32[2 * n + gi];
          const float d3 = qs[qq][3] - a.g.zs32[3 * n + gi];
          v = expf(lsv - 0.5f * (d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3));
        }
        kT[ii][qq] = v;
      }
      // L^{-T}[i0:i0+VI, j0:j0+VJ]
      for (int e = t; e < VI * VJ / 4; e += 256) {
        const int ii = e / (VJ / 4), jj = (e % (VJ / 4)) * 4;
        const int gi = i0 + ii, gj = j0 + jj;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gi < n) {
          const float* row = a.g.ilt32 + (size_t)gi * n;
          if (gj + 3 < n && ((n & 3) == 0)) {
            v = *reinterpret_cast<const float4*>(row + gj);
          } else {
            v.x = gj < n ? row[gj] : 0.f;
            v.y = gj + 1 < n ? row[gj + 1] : 0.f;
            v.z = gj + 2 < n ? row[gj + 2] : 0.f;
            v.w = gj + 3 < n ? row[gj + 3] : 0.f;
          }
        }
        *reinterpret_cast<float4*>(&Ls[ii][jj]) = v;
      }
      __syncthreads();
#pragma unroll 8
      for (int ii = 0; ii < VI; ++ii) {
        const float4 ka = *reinterpret_cast<const float4*>(&kT[ii][ty * 8]);
        const float4 kb = *reinterpret_cast<const float4*>(&kT[ii][ty * 8 + 4]);
        const float kk[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
        float l[4];
#pragma unroll
        for (int d = 0; d < 4; ++d) l[d] = Ls[ii][lane + 32 * d];
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
#pragma unroll
          for (int d = 0; d < 4; ++d) acc[qq][d] = fmaf(kk[qq], l[d], acc[qq][d]);
      }
    }
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      double p = 0.0;
#pragma unroll
      for (int d = 0; d < 4; ++d) p += (double)acc[qq][d] * (double)acc[qq][d];
      part[qq] += warp_sum(p);
    }
  }
  if (lane < 8) {
    double mine = 0.0;
#pragma unroll
    for (int qq = 0; qq < 8; ++qq)
      if (qq == lane) mine = part[qq];
    const long long qi = q0 + ty * 8 + lane;
    if (qi < a.KT) {
      double v = a.g.sv - mine;  // gp.cpp:187-191
      v = v > 0.0 ? v : 0.0;
      const double c = a.coef * v;
      a.trace[qi] = a.accumulate ? a.trace[qi] + c : c;
    }
  }
}

cudaError_t launch_tc_variance(const VarianceArgs& a, int mode, cudaStream_t st);  // kernels_tc.cu

cudaError_t launch_variance(const VarianceArgs& a, int path, cudaStream_t st) {
  if (a.KT <= 0) return cudaSuccess;
  if (path != 0) return launch_tc_variance(a, path == 4 ? 3 : path == 3 ? 2 : path == 2 ? 1 : 0, st);
  const long long blocks = (a.KT + VQ - 1) / VQ;
  variance_ffma_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

// -------------------------------------------------------------------------
// Reduction: tuple per block, last block combines (+ update/shift/diag).
int reduce_blocks_for(int K_local, int B, int num_sms, int T) {
  static const int forced = env_int("GPMPPI_REDUCE_BPR");
  // the last block of a robot stages every block tuple in shared memory (<= 160 KB)
  const int smem_cap = (int)((160 * 1024 / sizeof(double) - 2 * T) / (tuple_doubles(T) + 1));
  if (forced > 0) return forced < smem_cap ? forced : smem_cap;
  // blocks per robot: ~64 samples per block (measured: 148 blocks of 28 samples 34.8 us,
  // 64 blocks of 64 samples 28.6 us at K = 4096), at most one wave in total
  int b = (K_local + 63) / 64;
  const int cap = num_sms / (B < num_sms ? B : num_sms);
  if (b > cap) b = cap;
  if (b > smem_cap) b = smem_cap;
  return b < 1 ? 1 : b;
}

GPM_D void block_reduce_5(double v[5], double* red /*[32*5]*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < 5; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 5; ++i) red[w * 5 + i] = v[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 5; ++i) {
      double s = 0.0;
      for (int q = 0; q < nw; ++q) s += red[q * 5 + i];
      red[i] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 5; ++i) v[i] = red[i];
  __syncthreads();
}

// Apply a combined tuple: update + clamp (mppi.cpp:147-164), command (:430),
// shift (:166-173), diagnostics (:435-455). Executed by one block.
// Zero-copy completion word: the values land in pinned host memory (mapped), then -- after a
// system-scope fence -- word `seq_slot` receives the tick's sequence number, which the host
// polls instead of waiting on a copy and an event (latency of the command readback).
GPM_D void publish_host(double* host, const double* v, int nv, int seq_slot, double seq) {
  for (int i = 0; i < nv; ++i) host[i] = v[i];
  __threadfence_system();
  *reinterpret_cast<volatile double*>(host + seq_slot) = seq;
}

GPM_D void apply_tuple(const double* tup, int T, double lambda, double* nominal_seq,
                       const double lo[2], const double hi[2], double* out, long long K_total,
                       double* tmp /*2T*/, double* out_host = nullptr, double seq = 0.0) {
  const double Z = tup[1];
  for (int r = threadIdx.x; r < 2 * T; r += blockDim.x) {
    const double dv = Z > 0.0 ? tup[kTupleHead + r] / Z : 0.0;
    tmp[r] = clampd(nominal_seq[r] + dv, lo[r & 1], hi[r & 1]);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < 2 * T; r += blockDim.x) {
    const int k = r >> 1;
    nominal_seq[r] = k + 1 < T ? tmp[r + 2] : tmp[r];
  }
  if (threadIdx.x == 0) {
    const double m = tup[0], E2 = tup[2], H = tup[3], N = tup[4], C = tup[5];
    out[0] = tmp[0];
    out[1] = tmp[1];
    out[2] = N > 0.0 ? m : INFINITY;                                      // best_cost
    out[3] = N > 0.0 ? C / N : __longlong_as_double(0x7ff8000000000000LL);  // mean_cost
    out[4] = (Z > 0.0 && E2 > 0.0) ? (Z * Z) / E2 : 0.0;                   // ess = 1/Σw²
    out[5] = Z > 0.0 ? log(Z) + H / (lambda * Z) : 0.0;                    // -Σ w ln w
    out[6] = (double)K_total - N;                                           // nonfinite
    out[7] = N;
    if (out_host) publish_host(out_host, out, 8, BatchStrides::OUT - 1, seq);
  }
  __syncthreads();
}

// grid = B * bpr; block (b, j) reduces robot b's samples [j*per, (j+1)*per);
// the last block of each robot combines that robot's bpr tuples in block order.
// samples per pass-1 trace slab of the reduction (<= 96 KB of shared memory)
constexpr int kEpsDepth = 8;  // pass-3 noise loads in flight per thread

__global__ void __launch_bounds__(256, 1) reduce_kernel(const ReduceArgs a) {
  pdl_wait();
  if (threadIdx.x == 0) tl_stamp(5);
  pdl_trigger();
  // re-arm the rollout's query-progress words for the next tick: the co-resident variance
  // (the predecessor this grid waited for) has finished reading them
  if (a.progress)
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.progress_words;
         i += (long long)gridDim.x * blockDim.x)
      a.progress[i] = 0ull;
  extern __shared__ __align__(16) double dsm[];
  __shared__ double red[32 * 5];
  __shared__ unsigned int s_last;
#ifdef GPM_REDUCE_TRACE
  long long rt_[10];
  rt_[0] = clock64();
#define RTR(i) rt_[i] = clock64()
#else
#define RTR(i)
#endif
  const int T = a.T;
  const int b = blockIdx.x / a.bpr, j = blockIdx.x % a.bpr;
  const int per = (a.K_local + a.bpr - 1) / a.bpr;
  const long long base = (long long)b * a.K_local;  // robot-major sample slots
  const int b0 = j * per;
  const int b1 = min(a.K_local, b0 + per);
  const int W = tuple_doubles(T);
  const long long KT = query_slots(a.geom, a.B, T);  // per-group trace stride (item-major slots)
  const double* rt = a.x0 + (size_t)b * BatchStrides::X0;
  const double var_w = rt[5];
  const uint64_t key = (uint64_t)__double_as_longlong(rt[6]);
  double cg[kMaxGroups];  // Σ_o w(o)² of each group's outputs, computed with the weights on the host
#pragma unroll
  for (int g = 0; g < kMaxGroups; ++g) cg[g] = g < a.G ? a.tw[(size_t)b * BatchStrides::TW + BatchStrides::TW_COEF + g] : 0.0;
  // pass 1: costs (cost_mean + var_w * Σ_k Σ_g coef_g var_g), block min over finite.
  // Thread = sample; every sample sums its T traces in step order (mppi.cpp:34-49 combine,
  // costs.cpp:141). The traces are item-major (query_slot): for a fixed step the samples of
  // one rollout item are adjacent, so each step's loads coalesce across the warp; 8 steps
  // in flight per thread.
  double lmin = INFINITY;
  for (int s = b0 + (int)threadIdx.x; s < b1; s += blockDim.x) {
    const long long sl = base + s;
    double vsum = 0.0;
    if (a.var) {
      const long long q0 = query_slot(sl, 0, a.K_local, T, a.geom.spb, a.geom.chunks);
      const int spb = a.geom.spb;
      for (int g = 0; g < a.G; ++g) {
        const double* src = a.var + (size_t)g * KT + q0;
        double gsum = 0.0;
        int k = 0;
        for (; k + 16 <= T; k += 16) {  // 16 steps' loads in flight (HBM-bound at large K)
          double x[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) x[u] = __ldcs(src + (size_t)(k + u) * spb);
#pragma unroll
          for (int u = 0; u < 16; ++u) gsum += x[u];
        }
        for (; k < T; ++k) gsum += __ldcg(src + (size_t)k * spb);
        vsum += cg[g] * gsum;
      }
    }
    double c = a.cost_mean[sl];
    if (a.var) c += var_w * vsum;
    a.costs_out[sl] = c;
    if (isfinite(c)) lmin = fmin(lmin, c);
  }
  __syncthreads();  // the slab area is reused below
  lmin = warp_min(lmin);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lmin;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, red[w]);
    red[31 * 5] = m;
  }
  __syncthreads();
  const double mb = red[31 * 5];
  __syncthreads();
  RTR(1);
  // pass 2: e_s = exp(-(c - m_b)/lambda) (mppi.cpp:137-142) and scalar sums
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // Z, E2, H, N, C
  for (int s = b0 + threadIdx.x; s < b1; s += blockDim.x) {
    const double c = a.costs_out[base + s];
    double e = 0.0;
    if (isfinite(c)) {
      e = exp(-(c - mb) / a.lambda);
      v[0] += e;
      v[1] += e * e;
      v[2] += e * (c - mb);
      v[3] += 1.0;
      v[4] += c;
    }
    a.e_out[base + s] = e;
  }
  block_reduce_5(v, red);
  RTR(2);
  // pass 3: S[k][c] = Σ_s e_s eps[s][k][c]; thread = (k, slice)
  const int nsl = max(1, (int)blockDim.x / T);
  double* Ssl = dsm;  // [nsl][T][2]
  for (int idx = threadIdx.x; idx < T * nsl; idx += blockDim.x) {
    const int k = idx % T, sl = idx / T;
    double s0 = 0.0, s1 = 0.0;
    if (a.noise_mode == NOISE_INJECTED) {  // kEpsDepth samples' loads in flight per thread
      const double2* eps2 = reinterpret_cast<const double2*>(a.eps);
      for (int s = b0 + sl; s < b1; s += kEpsDepth * nsl) {
        double ev[kEpsDepth];
        double2 ep[kEpsDepth];
#pragma unroll
        for (int u = 0; u < kEpsDepth; ++u) {
          const int su = s + u * nsl;
          ev[u] = su < b1 ? __ldcg(a.e_out + base + su) : 0.0;
          ep[u] = su < b1 ? __ldcs(eps2 + (size_t)(base + su) * T + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kEpsDepth; ++u) {  // multiplied even when e = 0: a non-finite injected eps
          s0 += ev[u] * ep[u].x;       // poisons the update exactly as mppi.cpp:157-160 does
          s1 += ev[u] * ep[u].y;
        }
      }
    } else {
      for (int s = b0 + sl; s < b1; s += nsl) {
        const double e = a.e_out[base + s];
        if (e == 0.0) continue;
        double z1, z2;
        philox_gaussian_pair(key, (uint64_t)(a.s_begin + s), (uint32_t)k, &z1, &z2);
        s0 += e * (a.sv * z1);
        s1 += e * (a.sw * z2);
      }
    }
    Ssl[(sl * T + k) * 2] = s0;
    Ssl[(sl * T + k) * 2 + 1] = s1;
  }
  __syncthreads();
  RTR(3);
  double* mine = a.partials + (size_t)blockIdx.x * W;
  for (int r = threadIdx.x; r < 2 * T; r += blockDim.x) {
    double acc = 0.0;
    for (int sl = 0; sl < nsl; ++sl) acc += Ssl[sl * 2 * T + r];
    mine[kTupleHead + r] = acc;
  }
  if (threadIdx.x == 0) {
    mine[0] = v[3] > 0.0 ? mb : INFINITY;
    mine[1] = v[0];
    mine[2] = v[1];
    mine[3] = v[2];
    mine[4] = v[3];
    mine[5] = v[4];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(a.ticket + b, 1u) == (unsigned)a.bpr - 1);
  __syncthreads();
  RTR(4);
#ifdef GPM_REDUCE_TRACE
  if (threadIdx.x == 0 && (blockIdx.x == 0 || s_last))
    printf("reduce blk %d%s: pass1 %lld pass2 %lld pass3 %lld tuple+ticket %lld\n", blockIdx.x, s_last ? " (last)" : "",
           rt_[1] - rt_[0], rt_[2] - rt_[1], rt_[3] - rt_[2], rt_[4] - rt_[3]);
#endif
  if (!s_last) return;
  __threadfence();
  // last block of robot b: combine its block tuples in block order (heads staged in smem)
  double* tup = a.rank_tuple + (size_t)b * W;
  const double* parts = a.partials + (size_t)b * a.bpr * W;
  const int BP = a.bpr;
  double* pall = dsm;          // [BP][W] every block tuple (dsm holds >= BP*W + BP + 2T doubles)
  double* sc = dsm + (size_t)BP * W;  // [BP] rescale factors
  for (int i0 = threadIdx.x; i0 < BP * W; i0 += 8 * blockDim.x) {  // one coalesced sweep, 8 loads in flight
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      x[u] = i < BP * W ? __ldcg(parts + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < BP * W) pall[i] = x[u];
    }
  }
  __syncthreads();
  const int HW = W;  // head q at pall[q * W]
  double* heads = pall;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (threadIdx.x < 32) {  // global min of the block minima (exact in any order)
    double m = INFINITY;
    for (int q = lane; q < BP; q += 32) m = fmin(m, heads[q * HW]);
    m = warp_min(m);
    if (lane == 0) red[0] = m;
  }
  __syncthreads();
  RTR(5);
  const double m = red[0];
  for (int q = threadIdx.x; q < BP; q += blockDim.x)
    sc[q] = heads[q * HW + 4] > 0.0 ? exp(-(heads[q * HW] - m) / a.lambda) : 0.0;
  __syncthreads();
  if ((int)(threadIdx.x >> 5) == nw - 1) {  // last warp: the scalar sums, lane-strided then a fixed shuffle tree
    double Z = 0.0, E2 = 0.0, H = 0.0, N = 0.0, C = 0.0;
    for (int q = lane; q < BP; q += 32) {
      const double* p = heads + (size_t)q * HW;
      N += p[4];
      C += p[5];
      if (!(p[4] > 0.0)) continue;
      Z += sc[q] * p[1];
      E2 += sc[q] * sc[q] * p[2];
      H += sc[q] * (p[3] + (p[0] - m) * p[1]);
    }
    Z = warp_sum(Z);
    E2 = warp_sum(E2);
    H = warp_sum(H);
    N = warp_sum(N);
    C = warp_sum(C);
    if (lane == 0) {
      tup[0] = m;
      tup[1] = Z;
      tup[2] = E2;
      tup[3] = H;
      tup[4] = N;
      tup[5] = C;
      a.ticket[b] = 0u;  // re-arm for the next launch
    }
  }
  for (int r = threadIdx.x; r < 2 * T; r += blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < BP; ++q) acc = fma(sc[q], pall[(size_t)q * W + kTupleHead + r], acc);
    tup[kTupleHead + r] = acc;
  }
  __syncthreads();
  RTR(6);
  double* tmp = sc + BP;  // 2T doubles
  if (a.finish)
    apply_tuple(tup, T, a.lambda, a.nominal_seq + (size_t)b * BatchStrides::nom(T), a.lo, a.hi,
                a.out + (size_t)b * BatchStrides::OUT, a.K_total, tmp,
                a.out_host ? a.out_host + (size_t)b * BatchStrides::OUT : nullptr, rt[7]);
#ifdef GPM_REDUCE_TRACE
  RTR(7);
  if (threadIdx.x == 0)
    printf("reduce last: heads %lld combine+S %lld apply %lld\n", rt_[5] - rt_[4], rt_[6] - rt_[5], rt_[7] - rt_[6]);
#endif
  if (threadIdx.x == 0) tl_stamp(4);
}

cudaError_t launch_reduce(const ReduceArgs& a, int blocks, cudaStream_t st) {
  const int threads = 256;
  const int nsl = threads / a.T > 1 ? threads / a.T : 1;
  size_t smem = sizeof(double) * (size_t)nsl * a.T * 2;
  const size_t need = sizeof(double) * ((size_t)a.bpr * tuple_doubles(a.T) + a.bpr + 2 * a.T);
  if (smem < need) smem = need;
  cudaFuncSetAttribute(reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaError_t el = launch_pdl(reduce_kernel, dim3(blocks), dim3(threads), smem, st, a);
  if (el != cudaSuccess) return el;
  count_launch();
  return cudaGetLastError();
}

// Combine rank tuples (multi-GPU) and apply: one block.
__global__ void finish_kernel(const double* tuples, int n, int T, double lambda,
                              double* nominal_seq, double lo0, double lo1, double hi0, double hi1,
                              double* out, long long K_total, double* combined, double* out_host,
                              const double* x0_block) {
  extern __shared__ __align__(16) double tmp[];
  if (threadIdx.x == 0) combine_tuples(tuples, n, T, lambda, combined);
  __syncthreads();
  __threadfence_block();
  const double lo[2] = {lo0, lo1}, hi[2] = {hi0, hi1};
  apply_tuple(combined, T, lambda, nominal_seq, lo, hi, out, K_total, tmp, out_host, out_host ? x0_block[7] : 0.0);
}

cudaError_t launch_finish(const double* tuples, int n, int T, double lambda, double* nominal_seq,
                          const double lo[2], const double hi[2], double* out, long long K_total,
                          double* combined, cudaStream_t st, double* out_host, const double* x0_block) {
  finish_kernel<<<1, 128, sizeof(double) * 2 * T, st>>>(tuples, n, T, lambda, nominal_seq, lo[0],
                                                          lo[1], hi[0], hi[1], out, K_total,
                                                          combined, out_host, x0_block);
  count_launch();
  return cudaGetLastError();
}

// -------------------------------------------------------------------------
// FP64 single-query GP predict by one block (used by tightening and predict).
// Returns per-output mean (into mean[m]) and per-group variance (var_g[G]).
GPM_D void block_gp_predict(const ModelDev& M, const double q[4], double* kst /*n*/,
                            double* red /*>= 32*8*/, double* mean /*m*/, double* var_g) {
  const int n = M.n, ns = M.ns;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = 0; g < M.G; ++g) {
    const GroupDev& G = M.g[g];
    const double q0 = q[0] / G.ls[0], q1 = q[1] / G.ls[1], q2 = q[2] / G.ls[2], q3 = q[3] / G.ls[3];
    const double qn = -0.5 * (q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const double* p = G.pts;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double d = q0 * p[j] + q1 * p[ns + j] + q2 * p[2 * ns + j] + q3 * p[3 * ns + j] + qn + p[4 * ns + j];
      kst[j] = exp(d);  // each thread re-reads only its own entries below
    }
    for (int o0 = 0; o0 < G.n_out; o0 += kOutChunk) {  // k*.alpha, kOutChunk outputs per pass
      double acc[kOutChunk];
      for (int o = 0; o < kOutChunk; ++o) acc[o] = 0.0;
      const int no = min(kOutChunk, G.n_out - o0);
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double kj = kst[j];
        for (int o = 0; o < no; ++o) acc[o] = fma(kj, p[(5 + o0 + o) * ns + j], acc[o]);
      }
      for (int o = 0; o < no; ++o) {
        const double s = warp_sum(acc[o]);
        if (lane == 0) red[w * 8 + o] = s;
      }
      __syncthreads();
      if (threadIdx.x == 0)
        for (int o = 0; o < no; ++o) {
          double s = 0.0;
          for (int q2i = 0; q2i < nw; ++q2i) s += red[q2i * 8 + o];
          mean[G.out_idx[o0 + o]] = s;
        }
      __syncthreads();
    }
    // a_j = Σ_{i<=j} k_i L^{-T}[i][j]; ssq = Σ a_j^2
    double ssq = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double aj = 0.0;
      for (int i = 0; i <= j; ++i) aj = fma(kst[i], G.ilt64[(size_t)i * n + j], aj);
      ssq = fma(aj, aj, ssq);
    }
    ssq = warp_sum(ssq);
    if (lane == 0) red[w * 8] = ssq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q2i = 0; q2i < nw; ++q2i) s += red[q2i * 8];
      double v = G.sv - s;
      var_g[g] = v > 0.0 ? v : 0.0;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) predict_kernel(const ModelDev M, const double* q, long long S,
                                                      double* mean, double* var) {
  extern __shared__ __align__(16) double kst[];
  __shared__ double red[32 * 8];
  __shared__ double smean[kMaxGroups * kMaxOutPerGroup];
  __shared__ double svar[kMaxGroups];
  for (long long s = blockIdx.x; s < S; s += gridDim.x) {
    const double qq[4] = {q[s * 4], q[s * 4 + 1], q[s * 4 + 2], q[s * 4 + 3]};
    block_gp_predict(M, qq, kst, red, smean, svar);
    if (threadIdx.x == 0)
      for (int g = 0; g < M.G; ++g)
        for (int o = 0; o < M.g[g].n_out; ++o) {
          const int oi = M.g[g].out_idx[o];
          mean[s * M.m + oi] = smean[oi];
          var[s * M.m + oi] = svar[g];
        }
    __syncthreads();
  }
}

cudaError_t launch_predict(const ModelDev& m, const double* q, long long S, double* mean,
                           double* var, cudaStream_t st) {
  if (S <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * (size_t)m.n;
  cudaFuncSetAttribute(predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int blocks = S < 1184 ? (int)S : 1184;
  predict_kernel<<<blocks, 512, smem, st>>>(m, q, S, mean, var);
  count_launch();
  return cudaGetLastError();
}

// -------------------------------------------------------------------------
// Tightening pass (mppi.cpp:250-282 + uncertainty.cpp:75-116), FP64, in three
// launches. propagate_belief's mean update uses only the GP mean, never the
// covariance, so the belief-mean chain mu_0..mu_T is computed first (serial,
// one block), then every step's GP variance and Jacobian in parallel (one block
// per (step, group, column slice)), then the 5×5 covariance recursion and the
// thresholds (one warp).
// rows of L^{-1} per tightening-variance block: short slices (more, shorter blocks: the
// per-warp row loop is L2-latency bound) while the per-block k* recomputation is cheap
// (one robot only: with many robots the grid is already wide and 64-row slices recompute less)
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// a flag wait that outlives ~2 s is a protocol bug: trap instead of hanging the device
__device__ void spin_until_flag(const unsigned int* f, unsigned int at_least, const char* who) {
  // counter flags advance about once per chain step (~0.5 us): a waiter far behind sleeps in
  // proportion, so ~a thousand waiting blocks do not hammer one L2 line
  // relaxed polls (an acquire per poll invalidates L1 each time), one fence once it is seen
  for (unsigned it = 0, v; (v = ld_relaxed_u32(f)) < at_least; ++it) {
    const unsigned gap = at_least - v;
    __nanosleep(gap > 8u ? 2048u : 64u + 256u * (gap - 1u));
    if (it > (1u << 25)) {
      printf("%s: tightening flag wait timed out\n", who);
      __trap();
    }
  }
  __threadfence();  // acquire: the data published before the flag
}
#ifndef GPM_TIGHT_ROWS1
#define GPM_TIGHT_ROWS1 16
#endif
GPM_HD int tight_rows(int n, int B) { return (B == 1 && n <= 1024) ? GPM_TIGHT_ROWS1 : 64; }

// Belief-mean chain. The GP query of step k needs only (v_k, omega_k, u_k) and
// the lag update of (v, omega) is cheap, so the serial part carries (v, omega)
// only; theta is a cheap wrap recursion; the FP64 sincos / arc increments /
// Jacobians are then evaluated for all k in parallel and x, y accumulated in
// step order exactly as arc_advance does (dynamics.cpp:39-66).
#ifndef GPM_TMEAN_THREADS
#define GPM_TMEAN_THREADS 128
#endif
constexpr int TMEAN_THREADS = GPM_TMEAN_THREADS;
#ifndef GPM_PUB_SLEEP
#define GPM_PUB_SLEEP 32
#endif
template <int NO>
__global__ void __launch_bounds__(TMEAN_THREADS + 32, 1) tighten_mean_kernel(const TightenArgs a) {
  if (!a.tflags) pdl_trigger();  // pipelined: the variance grid is released after the reduction
  const int rb = blockIdx.x;  // robot
#ifdef GPM_TMEAN_TRACE
  const long long tk0 = clock64();
#endif
  const double* ax0 = a.x0 + (size_t)rb * BatchStrides::X0;
  double* atq = a.tq + (size_t)rb * 4 * a.T;
  double* atJ = a.tJ + (size_t)rb * 25 * a.T;
  double* atmu = a.tmu + (size_t)rb * 5 * (a.T + 1);
  extern __shared__ __align__(16) double tsm[];  // [2T nominal][T+1 v][T+1 w][T+1 th][T dx][T dy][pts]
  __shared__ double tw[kMaxTerrains];
  __shared__ double etab[32];
  if (threadIdx.x < 32) etab[threadIdx.x] = kExp2Frac[threadIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int T = a.T, n = a.model.n;
  double* nom = tsm;
  double* vv = nom + 2 * T;
  double* ww = vv + (T + 1);
  double* th = ww + (T + 1);
  double* dx = th + (T + 1);
  double* dy = dx + T;
  double* pts = dy + T + ((7 * T + 3) & 1);  // 16-byte aligned for the vectorised staging
  // model data and the host-staged terrain weights are ready before the predecessor
  // grid ends: staged ahead of griddepcontrol.wait (overlapping the reduction's tail)
  if (threadIdx.x < a.R) tw[threadIdx.x] = a.tw[(size_t)rb * BatchStrides::TW + threadIdx.x];
  if (a.model_kind == MODEL_GP) {  // vectorised staging of Z + terrain-combined alpha
    double* dst = pts;
    const int ns = a.model.ns;
    const double* rtw = a.tw + (size_t)rb * BatchStrides::TW;
    for (int g = 0; g < a.model.G; ++g) {
      const GroupDev& Gd = a.model.g[g];
      const double2* src = reinterpret_cast<const double2*>(Gd.pts);
      double2* d2 = reinterpret_cast<double2*>(dst);
#pragma unroll 10
      for (int i = threadIdx.x; i < 5 * ns / 2; i += blockDim.x) d2[i] = __ldg(src + i);
      // combine_terrains (mppi.cpp:34-49) folded into alpha, as in the rollout (load_robot_smem)
      for (int j = threadIdx.x; j < ns; j += blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        for (int o0 = 0; o0 < Gd.n_out; o0 += NO) {  // NO loads in flight (cold L2 after the rollout)
          double al[NO];
#pragma unroll
          for (int o = 0; o < NO; ++o)
            al[o] = o0 + o < Gd.n_out ? __ldg(Gd.pts + (size_t)(5 + o0 + o) * ns + j) : 0.0;
#pragma unroll
          for (int o = 0; o < NO; ++o) {
            if (o0 + o < Gd.n_out) {
              const int gi = Gd.out_idx[o0 + o];
              if (gi & 1)
                s1 = fma(rtw[gi >> 1], al[o], s1);
              else
                s0 = fma(rtw[gi >> 1], al[o], s0);
            }
          }
        }
        dst[5 * ns + j] = s0;
        dst[6 * ns + j] = s1;
      }
      dst += 7 * ns;
    }
  }
  pdl_wait();  // the nominal sequence comes from the reduction
  if (threadIdx.x == 0) tl_stamp(9);
  if (a.tflags) pdl_trigger();
  for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) nom[i] = a.nominal_seq[(size_t)rb * BatchStrides::nom(T) + i];
  if (threadIdx.x == 0) {
    vv[0] = ax0[3];
    ww[0] = ax0[4];
    th[0] = ax0[2];
  }
  __syncthreads();
  const double av = a.nom.dt / a.nom.tau_v, aw = a.nom.dt / a.nom.tau_omega;
  // serial (v, omega) chain with the GP mean (mppi.cpp:220-233). The warps split the
  // n points; every warp reduces the per-warp partials itself (double-buffered), so a
  // step costs one block barrier. q/l uses reciprocal lengthscales (<= 1 ulp from the
  // reference's division) to keep FP64 divides off the serial path.
  __shared__ __align__(16) double red[2][kMaxGroups][TMEAN_THREADS / 32][2];  // [parity][group][warp][v, omega]
  __shared__ double gil[kMaxGroups][4];  // reciprocal lengthscales
  // pipelined (a.tflags): warp TMEAN_THREADS / 32 publishes each step's query (and raises the
  // query counter, flag 0) while the chain warps run on: its fences stay off the serial path
  __shared__ volatile int prog;  // chain steps done (thread 0, after vv / ww)
  // pipelined (a.tflags): the warp after the chain's publishes, per batch of finished steps, the
  // queries (flag 0), then the Jacobians and belief means (flag 1) -- tighten_cov_pipe_kernel
  // and the variance grid, launched after this kernel, consume them step by step
  const bool pub = a.tflags != nullptr && threadIdx.x >= TMEAN_THREADS;
  if (threadIdx.x == 0) prog = 0;
  const int ns = a.model.ns;
  const int G = a.model_kind == MODEL_GP ? a.model.G : 0;
  if (threadIdx.x < 4 * G) gil[threadIdx.x >> 2][threadIdx.x & 3] = 1.0 / a.model.g[threadIdx.x >> 2].ls[threadIdx.x & 3];
  __syncthreads();
  double v = vv[0], om = ww[0];
#ifdef GPM_TMEAN_TRACE
  const long long tk1 = clock64();
  long long tr[8] = {};
#define TRC(i) if (k == 5) tr[i] = clock64()
#else
#define TRC(i)
#endif
  // One kernel group and n <= 4 * TMEAN_THREADS (configs 1, 2, 4, 5): every thread keeps its
  // four points' Z / alpha in registers for the whole chain, and the control-dependent part of
  // each exponent, q2 z2 + q3 z3 + zn - (q2^2 + q3^2)/2, is formed for step k+1 while step k's
  // partial sums cross the barrier -- the serial path per step is 2 FMAs + the exp per point.
  const bool reg_path = G == 1 && n <= 4 * TMEAN_THREADS;
  double rz0[4], rz1[4], rz2[4], rz3[4], rzn[4], rav[4], raw[4], e_cur[4];
  if (reg_path) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = threadIdx.x + i * TMEAN_THREADS;
      const bool in = j < n;
      rz0[i] = in ? pts[j] : 0.0;
      rz1[i] = in ? pts[ns + j] : 0.0;
      rz2[i] = in ? pts[2 * ns + j] : 0.0;
      rz3[i] = in ? pts[3 * ns + j] : 0.0;
      rzn[i] = in ? pts[4 * ns + j] : -1e300;  // exp_tab flushes to 0
      rav[i] = in ? pts[5 * ns + j] : 0.0;
      raw[i] = in ? pts[6 * ns + j] : 0.0;
    }
    const double q2 = nom[0] * gil[0][2], q3 = nom[1] * gil[0][3];
    const double qu = -0.5 * (q2 * q2 + q3 * q3);
#pragma unroll
    for (int i = 0; i < 4; ++i) e_cur[i] = fma(q2, rz2[i], fma(q3, rz3[i], rzn[i] + qu));
  }
  if (pub) {
    if (a.cmd_host && lane == 0) {  // the reduction's command and diagnostics into the mapped words
      double o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = __ldcg(a.cmd_dev + i);
      publish_host(a.cmd_host, o, 8, BatchStrides::OUT - 1, a.x0[7]);
    }
    // the publisher warp walks the chain's steps as they complete (convergent): per batch of
    // newly known steps, lane 0 advances the heading recursion, one lane per step evaluates the
    // arc increment and the Jacobian (as the sequential tail below), lane 0 writes the queries,
    // the belief means (positions summed in step order) and raises the query counter; after
    // the last step, the final belief mean and flag 1
    double px = ax0[0], py = ax0[1];  // lane 0: position prefix sums
    double t = th[0];                 // lane 0: heading recursion
    for (int k = 0; k < T;) {
      int done;
      for (unsigned it = 0; (done = prog) < k; ++it) {  // sleep between polls: the chain shares this scheduler
        __nanosleep(GPM_PUB_SLEEP);
        if (it > (1u << 27)) __trap();
      }
      done = __shfl_sync(0xffffffffu, done, 0);
      const int k1 = done + 1 < T ? done + 1 : T;  // query k = (v_k, omega_k, u_k): known once step k-1 is done
      if (lane == 0) {  // the queries first: the variance blocks of these steps wait for them
        for (int kk = k; kk < k1; ++kk) {
          atq[kk * 4 + 0] = vv[kk];
          atq[kk * 4 + 1] = ww[kk];
          atq[kk * 4 + 2] = nom[2 * kk];
          atq[kk * 4 + 3] = nom[2 * kk + 1];
        }
        st_release_u32(a.tflags, (unsigned)k1);  // queries [0, k1) are out (release: lane 0's stores first)
      }
      if (lane == 0)
        for (int kk = k; kk < k1; ++kk) {  // arc_advance: theta = wrap(theta + omega dt)
          t = t + ww[kk] * a.nom.dt;
          if (!(t > -kPi && t <= kPi)) t = wrap_angle_fast(t);
          th[kk + 1] = t;
        }
      __syncwarp();
      for (int kk = k + lane; kk < k1; kk += 32) {
        const double m0[5] = {0.0, 0.0, th[kk], vv[kk], ww[kk]};
        double s0, c0;
        sincos(th[kk], &s0, &c0);
        double x = 0.0, y = 0.0, t2 = th[kk];
        arc_advance(x, y, t2, vv[kk], 0.0, ww[kk], a.nom.dt, s0, c0);
        dx[kk] = x;
        dy[kk] = y;
        double J[25];
        jacobian_nominal(m0, a.nom, J);
        for (int i = 0; i < 25; ++i) atJ[kk * 25 + i] = J[i];
      }
      __syncwarp();
      if (lane == 0) {
        for (int kk = k; kk < k1; ++kk) {  // belief mean before step kk
          atmu[kk * 5 + 0] = px;
          atmu[kk * 5 + 1] = py;
          atmu[kk * 5 + 2] = th[kk];
          atmu[kk * 5 + 3] = vv[kk];
          atmu[kk * 5 + 4] = ww[kk];
          px += dx[kk];
          py += dy[kk];
        }
      }
      __syncwarp();  // every lane's Jacobians before lane 0's release
      if (lane == 0) st_release_u32(a.tflags + 1, (unsigned)k1);  // J_k and mu_k out for k < k1
      k = k1;
    }
    for (unsigned it = 0; prog < T; ++it)  // the final belief mean needs the last step's (v, omega)
      if (it > (1u << 28)) __trap();
    if (lane == 0) {
      atmu[T * 5 + 0] = px;
      atmu[T * 5 + 1] = py;
      atmu[T * 5 + 2] = th[T];
      atmu[T * 5 + 3] = vv[T];
      atmu[T * 5 + 4] = ww[T];
    }
    if (lane == 0) {
      st_release_u32(a.tflags + 1, (unsigned)T + 1u);  // and the final belief mean
      tl_stamp(8);
    }
  } else
  for (int k = 0; k < T; ++k) {
    TRC(0);
    const double u0 = nom[2 * k], u1 = nom[2 * k + 1];
    double c0 = 0.0, c1 = 0.0;
    if (reg_path) {
      const double q0 = v * gil[0][0], q1 = om * gil[0][1];
      const double qv = -0.5 * (q0 * q0 + q1 * q1);
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double kj = exp_tab(fma(q0, rz0[i], fma(q1, rz1[i], e_cur[i] + qv)), etab);
        acc0 = fma(kj, rav[i], acc0);
        acc1 = fma(kj, raw[i], acc1);
      }
      TRC(1);
      {  // transpose-reduce the two sums across the warp (5 shuffles), as below
        const bool b4 = lane & 16;
        double y = (b4 ? acc1 : acc0) + __shfl_xor_sync(0xffffffffu, b4 ? acc0 : acc1, 16);
        y += __shfl_xor_sync(0xffffffffu, y, 8);
        y += __shfl_xor_sync(0xffffffffu, y, 4);
        y += __shfl_xor_sync(0xffffffffu, y, 2);
        y += __shfl_xor_sync(0xffffffffu, y, 1);
        if ((lane & 15) == 0) red[k & 1][0][w][lane >> 4] = y;
      }
      TRC(2);
      if (k + 1 < T) {  // next step's control part, in the shadow of the barrier
        const double q2 = nom[2 * k + 2] * gil[0][2], q3 = nom[2 * k + 3] * gil[0][3];
        const double qu = -0.5 * (q2 * q2 + q3 * q3);
#pragma unroll
        for (int i = 0; i < 4; ++i) e_cur[i] = fma(q2, rz2[i], fma(q3, rz3[i], rzn[i] + qu));
      }
      asm volatile("bar.sync 1, %0;" ::"n"(TMEAN_THREADS) : "memory");  // the chain warps
      TRC(3);
      double2 pr[TMEAN_THREADS / 32];
#pragma unroll
      for (int q = 0; q < TMEAN_THREADS / 32; ++q) pr[q] = *reinterpret_cast<const double2*>(&red[k & 1][0][q][0]);
      double x0 = pr[0].x, x1 = pr[0].y;
#pragma unroll
      for (int q = 1; q < TMEAN_THREADS / 32; ++q) {
        x0 += pr[q].x;
        x1 += pr[q].y;
      }
      c0 = x0;
      c1 = x1;
    } else if (G > 0) {
      const double* p = pts;
      for (int g = 0; g < G; ++g) {
        const double q0 = v * gil[g][0], q1 = om * gil[g][1];
        const double q2 = u0 * gil[g][2], q3 = u1 * gil[g][3];
        const double qn = -0.5 * (q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
        double acc0 = 0.0, acc1 = 0.0;  // terrain-combined v / omega means
        // four points per round with their exponentials side by side
        for (int j0 = threadIdx.x; j0 < n; j0 += 4 * TMEAN_THREADS) {
          double kj[4], av[4], aw[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int j = j0 + i * TMEAN_THREADS;
            const bool in = j < n;
            const int jc = in ? j : j0;
            const double d = fma(q0, p[jc], fma(q1, p[ns + jc], fma(q2, p[2 * ns + jc], fma(q3, p[3 * ns + jc], qn + p[4 * ns + jc]))));
            kj[i] = exp_tab(d, etab);
            av[i] = in ? p[5 * ns + jc] : 0.0;
            aw[i] = in ? p[6 * ns + jc] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc0 = fma(kj[i], av[i], acc0);
            acc1 = fma(kj[i], aw[i], acc1);
          }
        }
        TRC(1);
        {  // transpose-reduce the two sums across the warp (5 shuffles): lanes 0-15
           // end with the v total, lanes 16-31 with the omega total
          const bool b4 = lane & 16;
          double y = (b4 ? acc1 : acc0) + __shfl_xor_sync(0xffffffffu, b4 ? acc0 : acc1, 16);
          y += __shfl_xor_sync(0xffffffffu, y, 8);
          y += __shfl_xor_sync(0xffffffffu, y, 4);
          y += __shfl_xor_sync(0xffffffffu, y, 2);
          y += __shfl_xor_sync(0xffffffffu, y, 1);
          if ((lane & 15) == 0) red[k & 1][g][w][lane >> 4] = y;
        }
        TRC(2);
        p += (size_t)7 * ns;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(TMEAN_THREADS) : "memory");  // the chain warps
      TRC(3);
      for (int g = 0; g < G; ++g) {
        // every thread sums the per-warp partials in warp order (identical bits everywhere)
        double2 pr[TMEAN_THREADS / 32];  // 16-byte loads, all issued before the sums
#pragma unroll
        for (int q = 0; q < TMEAN_THREADS / 32; ++q) pr[q] = *reinterpret_cast<const double2*>(&red[k & 1][g][q][0]);
        double x0 = pr[0].x, x1 = pr[0].y;
#pragma unroll
        for (int q = 1; q < TMEAN_THREADS / 32; ++q) {
          x0 += pr[q].x;
          x1 += pr[q].y;
        }
        c0 += x0;
        c1 += x1;
      }
    }
    TRC(4);
    if (threadIdx.x == 0 && !a.tflags) {
      atq[k * 4 + 0] = v;
      atq[k * 4 + 1] = om;
      atq[k * 4 + 2] = u0;
      atq[k * 4 + 3] = u1;
    }
    v = v + av * (u0 - v) + c0;  // step_nominal lag (dynamics.cpp:63-64) + correction mean
    om = om + aw * (u1 - om) + c1;
#ifdef GPM_TMEAN_TRACE
    if (k == 5 && (threadIdx.x & 31) == 0) {
      const long long t5 = clock64();
      printf("tmean w%d: loop %lld shfl %lld bar %lld sum %lld upd %lld total %lld (v %.3e)\n", (int)(threadIdx.x >> 5),
             tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3], t5 - tr[4], t5 - tr[0], v);
    }
#endif
    if (threadIdx.x == 0) {
      vv[k + 1] = v;
      ww[k + 1] = om;
      if (a.tflags) {
        __threadfence_block();
        prog = k + 1;
      }
    }
  }
  if (threadIdx.x == 0) tl_stamp(6);
  __syncthreads();
#ifdef GPM_TMEAN_TRACE
  const long long tk2 = clock64();
#endif
  if (!a.tflags) {  // sequential tail (the publisher warp did this step by step when pipelined)
  if (threadIdx.x == 0) {  // heading recursion (arc_advance: theta = wrap(theta + omega dt))
    double t = th[0];
    for (int k0 = 0; k0 < T; k0 += 8) {  // omega read 8 steps ahead; wrap only off (-pi, pi]
      double wv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) wv[i] = k0 + i < T ? ww[k0 + i] : 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (k0 + i < T) {
          t = t + wv[i] * a.nom.dt;
          if (!(t > -kPi && t <= kPi)) t = wrap_angle_fast(t);
          th[k0 + i + 1] = t;
        }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < T; k += blockDim.x) {  // arc increments + Jacobians, parallel in k
    const double m0[5] = {0.0, 0.0, th[k], vv[k], ww[k]};
    double s0, c0;
    sincos(th[k], &s0, &c0);
    double x = 0.0, y = 0.0, t2 = th[k];
    arc_advance(x, y, t2, vv[k], 0.0, ww[k], a.nom.dt, s0, c0);
    dx[k] = x;
    dy[k] = y;
    double J[25];
    jacobian_nominal(m0, a.nom, J);
    for (int i = 0; i < 25; ++i) atJ[k * 25 + i] = J[i];
  }
  __syncthreads();
  for (int k = threadIdx.x; k <= T; k += blockDim.x) {  // heading / speeds of every belief mean
    atmu[k * 5 + 2] = th[k];
    atmu[k * 5 + 3] = vv[k];
    atmu[k * 5 + 4] = ww[k];
  }
  if (threadIdx.x == 0) {  // positions: prefix sum in step order, increments read 8 ahead
    double x = ax0[0], y = ax0[1];
    atmu[0] = x;
    atmu[1] = y;
    for (int k0 = 0; k0 < T; k0 += 8) {
      double ddx[8], ddy[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        ddx[i] = k0 + i < T ? dx[k0 + i] : 0.0;
        ddy[i] = k0 + i < T ? dy[k0 + i] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (k0 + i < T) {
          x += ddx[i];
          y += ddy[i];
          atmu[(k0 + i + 1) * 5 + 0] = x;
          atmu[(k0 + i + 1) * 5 + 1] = y;
        }
    }
  }
  }

#ifdef GPM_TMEAN_TRACE
  if (threadIdx.x == 0) {
    const long long tk3 = clock64();
    printf("tmean kernel: staging %lld chain %lld tail %lld total %lld\n", tk1 - tk0, tk2 - tk1, tk3 - tk2, tk3 - tk0);
  }
#endif
}

// grid (ceil(n / tight_rows(n, B)), G*B, T): partial ||L^{-1} k*||^2 over a slice of rows of
// L^{-1} (x = slice fastest, so the blocks are scheduled step by step, the order in which the
// pipelined pass releases them). One warp per row: a_j = sum_{i<=j} k_i L^{-1}[j][i] with the lanes striding
// the contiguous row (coalesced), then a_j^2 (gp.cpp:184-191).
__global__ void __launch_bounds__(256) tighten_var_kernel(const TightenArgs a) {
  if (threadIdx.x == 0) tl_stamp(11);
  if (a.tflags) {  // pipelined: start when the mean chain's queries are out (flag 0)
    pdl_trigger();
    if (threadIdx.x == 0) spin_until_flag(a.tflags, (unsigned)blockIdx.z + 1u, "tighten_var_kernel");
    if (threadIdx.x == 0 && blockIdx.z == gridDim.z - 1) {
      tl_stamp(21);
      tl_stamp(20);
    }
    if (threadIdx.x == 0 && blockIdx.z == 0) tl_stamp(29);
    __syncthreads();
  } else {
    pdl_wait();
    pdl_trigger();
  }
  extern __shared__ __align__(16) double kst[];
  __shared__ double red[8];
  const int k = blockIdx.z, g = blockIdx.y % a.model.G, rb = blockIdx.y / a.model.G, c = blockIdx.x;
  const int n = a.model.n;
  if (a.model_kind != MODEL_GP) return;
  const GroupDev& G = a.model.g[g];
  const double* q = a.tq + (size_t)rb * 4 * a.T + k * 4;
  const double q0 = q[0] / G.ls[0], q1 = q[1] / G.ls[1], q2 = q[2] / G.ls[2], q3 = q[3] / G.ls[3];
  const double qn = -0.5 * (q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
  const int rows = tight_rows(n, a.B);
  const int j0 = c * rows;
  const int jend = min(n, j0 + rows);
  const double* p = G.pts;
  const int ns = a.model.ns;
  __shared__ double etab[32];
  if (threadIdx.x < 32) etab[threadIdx.x] = kExp2Frac[threadIdx.x];
  __syncthreads();
  for (int i = threadIdx.x; i < jend; i += blockDim.x)  // columns i <= j only
    kst[i] = exp_tab(fma(q0, p[i], fma(q1, p[ns + i], fma(q2, p[2 * ns + i], fma(q3, p[3 * ns + i], qn + p[4 * ns + i])))), etab);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double ssq = 0.0;
  for (int j = j0 + w; j < jend; j += 8) {
    const double* row = G.linv64 + (size_t)j * n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = lane;
    for (; i + 480 <= j; i += 512) {  // sixteen independent loads in flight per lane
      double r[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) r[u] = __ldg(row + i + 32 * u);
#pragma unroll
      for (int u = 0; u < 16; u += 4) {
        a0 = fma(kst[i + 32 * u], r[u], a0);
        a1 = fma(kst[i + 32 * (u + 1)], r[u + 1], a1);
        a2 = fma(kst[i + 32 * (u + 2)], r[u + 2], a2);
        a3 = fma(kst[i + 32 * (u + 3)], r[u + 3], a3);
      }
    }
    {  // the remaining < 16 column strides of the row, loads predicated, all in flight
      double r[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) r[u] = i + 32 * u <= j ? __ldg(row + i + 32 * u) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; u += 4) {
        if (i + 32 * u <= j) a0 = fma(kst[i + 32 * u], r[u], a0);
        if (i + 32 * (u + 1) <= j) a1 = fma(kst[i + 32 * (u + 1)], r[u + 1], a1);
        if (i + 32 * (u + 2) <= j) a2 = fma(kst[i + 32 * (u + 2)], r[u + 2], a2);
        if (i + 32 * (u + 3) <= j) a3 = fma(kst[i + 32 * (u + 3)], r[u + 3], a3);
      }
    }
    const double aj = warp_sum((a0 + a1) + (a2 + a3));
    ssq = fma(aj, aj, ssq);
  }
  if (lane == 0) red[w] = ssq;
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += red[i];
    a.tvar_part[(((size_t)rb * a.T + k) * a.model.G + g) * gridDim.x + c] = s;
    if (k == 0) {
      tl_stamp(31);
      tl_stamp(14);
    }
    s_last = 0;
    if (a.tflags) {  // pipelined: the step's last slice block also combines the step (cv_k)
      unsigned prev;  // acq_rel: releases this slice's partial, acquires every earlier slice's
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.tflags + 2 + k) : "memory");
      s_last = prev == (unsigned)(gridDim.x * a.model.G) - 1u;
    }
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {  // warp 0: every slice in flight at once, summed in split order
    if (k == 0 && lane == 0) tl_stamp(27);
    __syncwarp();
    double vg[kMaxGroups];
#pragma unroll
    for (int gg = 0; gg < kMaxGroups; ++gg) vg[gg] = 0.0;
    for (int gg = 0; gg < a.model.G; ++gg) {
      const double* pv = a.tvar_part + ((size_t)k * a.model.G + gg) * gridDim.x;
      double sum = 0.0;
      for (int c0 = 0; c0 < (int)gridDim.x; c0 += 32) {
        const double x = c0 + lane < (int)gridDim.x ? __ldcg(pv + c0 + lane) : 0.0;
        const int cn = (int)gridDim.x - c0 < 32 ? (int)gridDim.x - c0 : 32;
        for (int cc = 0; cc < cn; ++cc) sum += __shfl_sync(0xffffffffu, x, cc);
      }
      const double v = a.model.g[gg].sv - sum;
      vg[gg] = v > 0.0 ? v : 0.0;
    }
    if (lane == 0) {
      double c0 = 0.0, c1 = 0.0;  // ensemble_combine's Σ w² v per channel (gp.cpp:380-386)
      for (int i = 0; i < a.R; ++i) {
        const double wi = a.tw[i];
        int g0 = 0, g1 = 0;
        for (int gg = 0; gg < a.model.G; ++gg)
          for (int o = 0; o < a.model.g[gg].n_out; ++o) {
            if (a.model.g[gg].out_idx[o] == 2 * i) g0 = gg;
            if (a.model.g[gg].out_idx[o] == 2 * i + 1) g1 = gg;
          }
        double v0 = vg[0], v1 = vg[0];
#pragma unroll
        for (int gg = 1; gg < kMaxGroups; ++gg) {
          v0 = g0 == gg ? vg[gg] : v0;
          v1 = g1 == gg ? vg[gg] : v1;
        }
        c0 += wi * wi * v0;
        c1 += wi * wi * v1;
      }
      a.tcv[2 * k] = c0;
      a.tcv[2 * k + 1] = c1;
      st_release_u32(a.tflags + 2 + k, 0x40000000u);  // cv_k is out (release: the stores above first)
      if (k == 0) tl_stamp(25);
    }
  }
  if (threadIdx.x == 0) tl_stamp(10);
}

// One step of the belief covariance recursion Σ' = J Σ Jᵀ + diag(0,0,0,cv0,cv1)
// (uncertainty.cpp:83-87) in registers. jacobian_nominal (dynamics.cpp:68-98) is structurally
// sparse, J = [1 0 a b c; 0 1 d e f; 0 0 1 0 g; 0 0 0 h 0; 0 0 0 0 i] (j[0..8] = a..i), so a
// step is P = JΣ (3-FMA rows) then the 15 upper entries of PJᵀ: a 6-FMA-deep chain. Σ stays
// exactly symmetric, so the reference's symmetrisation is the identity here. s[15] holds the
// upper triangle row by row (00 01 02 03 04 11 12 13 14 22 23 24 33 34 44); Sk gets all 25.
GPM_D void cov_step(const double j[9], double cv0, double cv1, double s[15], double* Sk) {
  const double ja = j[0], jb = j[1], jc = j[2], jd = j[3], je = j[4], jf = j[5], jg = j[6], jh = j[7], ji = j[8];
  const double s00 = s[0], s01 = s[1], s02 = s[2], s03 = s[3], s04 = s[4], s11 = s[5], s12 = s[6], s13 = s[7];
  const double s14 = s[8], s22 = s[9], s23 = s[10], s24 = s[11], s33 = s[12], s34 = s[13], s44 = s[14];
  const double p00 = fma(jc, s04, fma(jb, s03, fma(ja, s02, s00)));
  const double p01 = fma(jc, s14, fma(jb, s13, fma(ja, s12, s01)));
  const double p02 = fma(jc, s24, fma(jb, s23, fma(ja, s22, s02)));
  const double p03 = fma(jc, s34, fma(jb, s33, fma(ja, s23, s03)));
  const double p04 = fma(jc, s44, fma(jb, s34, fma(ja, s24, s04)));
  const double p11 = fma(jf, s14, fma(je, s13, fma(jd, s12, s11)));
  const double p12 = fma(jf, s24, fma(je, s23, fma(jd, s22, s12)));
  const double p13 = fma(jf, s34, fma(je, s33, fma(jd, s23, s13)));
  const double p14 = fma(jf, s44, fma(je, s34, fma(jd, s24, s14)));
  const double p22 = fma(jg, s24, s22), p23 = fma(jg, s34, s23), p24 = fma(jg, s44, s24);
  const double p33 = jh * s33, p34 = jh * s34, p44 = ji * s44;
  s[0] = fma(jc, p04, fma(jb, p03, fma(ja, p02, p00)));
  s[1] = fma(jf, p04, fma(je, p03, fma(jd, p02, p01)));
  s[2] = fma(jg, p04, p02);
  s[3] = jh * p03;
  s[4] = ji * p04;
  s[5] = fma(jf, p14, fma(je, p13, fma(jd, p12, p11)));
  s[6] = fma(jg, p14, p12);
  s[7] = jh * p13;
  s[8] = ji * p14;
  s[9] = fma(jg, p24, p22);
  s[10] = jh * p23;
  s[11] = ji * p24;
  s[12] = fma(jh, p33, cv0);
  s[13] = ji * p34;
  s[14] = fma(ji, p44, cv1);
  Sk[0] = s[0], Sk[1] = s[1], Sk[2] = s[2], Sk[3] = s[3], Sk[4] = s[4];
  Sk[5] = s[1], Sk[6] = s[5], Sk[7] = s[6], Sk[8] = s[7], Sk[9] = s[8];
  Sk[10] = s[2], Sk[11] = s[6], Sk[12] = s[9], Sk[13] = s[10], Sk[14] = s[11];
  Sk[15] = s[3], Sk[16] = s[7], Sk[17] = s[10], Sk[18] = s[12], Sk[19] = s[13];
  Sk[20] = s[4], Sk[21] = s[8], Sk[22] = s[11], Sk[23] = s[13], Sk[24] = s[14];
}
// tighten_lane_radius (uncertainty.cpp:90-96) from Σ's (x, y) block
GPM_D double lane_radius(const double* Sk, double half_width, double chi2) {
  const double c00 = Sk[0], c01 = Sk[1], c10 = Sk[5], c11 = Sk[6];
  const double half_tr = 0.5 * (c00 + c11);
  const double disc = 0.25 * (c00 - c11) * (c00 - c11) + c01 * c10;
  double lm = half_tr + sqrt(disc > 0.0 ? disc : 0.0);
  lm = lm > 0.0 ? lm : 0.0;
  return half_width - sqrt(chi2 * lm);
}
// tighten_obstacle_distance (uncertainty.cpp:98-116): margin d - d̄ of one obstacle; *tight = d̄
GPM_D double obstacle_margin(const double* Sk, double mx, double my, const double obs[3], double z, double* tight) {
  const double c00 = Sk[0], c01 = Sk[1], c10 = Sk[5], c11 = Sk[6];
  const double dx = mx - obs[0], dy = my - obs[1];
  const double dist = sqrt(dx * dx + dy * dy);
  double d, n0, n1;
  if (dist < 1e-12) {
    n0 = 1.0;
    n1 = 0.0;
    d = -obs[2];
  } else {
    n0 = dx / dist;
    n1 = dy / dist;
    d = dist - obs[2];
  }
  const double cn0 = c00 * n0 + c01 * n1, cn1 = c10 * n0 + c11 * n1;
  double dv = n0 * cn0 + n1 * cn1;
  dv = dv > 0.0 ? dv : 0.0;
  const double dbar = d - z * sqrt(dv);
  *tight = dbar;
  return d - dbar;
}

// 256 threads stage J / mu / the per-step correction variances, warp 0 runs the
// serial recursion Σ_{k+1} = J Σ Jᵀ + diag(0,0,0,cv0,cv1) (symmetrised), then all
// threads evaluate r̄_k and the margins in parallel.
__global__ void __launch_bounds__(256, 1) tighten_cov_kernel(const TightenArgs a, int nsplit) {
  // with a GP the predecessor is the variance grid and the mean kernel's J / belief
  // means are already complete; without one the mean kernel is the predecessor
  if (a.model_kind != MODEL_GP) pdl_wait();
  pdl_trigger();
  const int rb = blockIdx.x;  // robot
#ifdef GPM_TCOV_TRACE
  long long ct[6];
  ct[0] = clock64();
#endif
  const double* atJ = a.tJ + (size_t)rb * 25 * a.T;
  const double* atmu = a.tmu + (size_t)rb * 5 * (a.T + 1);
  const double* atvar = a.tvar_part + (size_t)rb * a.T * (a.model_kind == MODEL_GP ? a.model.G : 1) * nsplit;
  const double* atw = a.tw + (size_t)rb * BatchStrides::TW;
  double* ahcov = a.horizon_cov + (size_t)rb * 25 * a.T;
  double* arbar = a.r_bar + (size_t)rb * BatchStrides::rbar(a.T);
  double* amarg = a.margins + (size_t)rb * BatchStrides::marg(a.T);
  extern __shared__ __align__(16) double csm[];  // [T][25] J, [T][2] cv, [T+1][5] mu
  __shared__ int infeasible;
  __shared__ int gof[2 * kMaxTerrains];  // kernel group of each GP output
  const int l = threadIdx.x;
  const int nt = blockDim.x;
  const TaskDev& t = a.task[rb];
  const int T = a.T;
  double* Js = csm;
  double* cvs = csm + 25 * T;
  double* mus = cvs + 2 * T;
  const int G = a.model_kind == MODEL_GP ? a.model.G : 0;
  if (l == 0) {
    infeasible = 0;
    for (int g = 0; g < G; ++g)
      for (int o = 0; o < a.model.g[g].n_out; ++o) gof[a.model.g[g].out_idx[o]] = g;
  }
  // J and the belief means are written by tighten_mean_kernel, two launches back: PTX
  // guarantees their visibility only after this grid's own griddepcontrol.wait, so the
  // staging follows it (it does not rely on the variance grid's wait-before-trigger order)
  pdl_wait();
  if (l == 0) tl_stamp(13);
  for (int i = l; i < 25 * T; i += nt) Js[i] = atJ[i];
  for (int i = l; i < 5 * (T + 1); i += nt) mus[i] = atmu[i];
  __syncthreads();
  // per-step combined correction variance (gp.cpp:187-191 + ensemble_combine gp.cpp:380-386)
  for (int k = l; k < T; k += nt) {
    double c0 = 0.0, c1 = 0.0;
    if (G > 0) {
      double vg[kMaxGroups];
#pragma unroll
      for (int g = 0; g < kMaxGroups; ++g) {
        double v = 0.0;
        if (g < G) {
          const double* pv = atvar + ((size_t)k * G + g) * nsplit;
          double s = 0.0;
          int c = 0;
          for (; c + 8 <= nsplit; c += 8) {  // eight loads in flight, summed in split order
            double x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = pv[c + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) s += x[u];
          }
          for (; c < nsplit; ++c) s += pv[c];
          v = a.model.g[g].sv - s;
        }
        vg[g] = v > 0.0 ? v : 0.0;
      }
      for (int i = 0; i < a.R; ++i) {
        const double wi = atw[i];
        const int g0 = gof[2 * i], g1 = gof[2 * i + 1];
        double v0 = vg[0], v1 = vg[0];  // register select (no local-memory indexing)
#pragma unroll
        for (int g = 1; g < kMaxGroups; ++g) {
          v0 = g0 == g ? vg[g] : v0;
          v1 = g1 == g ? vg[g] : v1;
        }
        c0 += wi * wi * v0;
        c1 += wi * wi * v1;
      }
    }
    cvs[2 * k] = c0;
    cvs[2 * k + 1] = c1;
  }
  double* Ss = mus + 5 * (T + 1);  // [T][25] propagated covariances
  __syncthreads();
#ifdef GPM_TCOV_TRACE
  ct[1] = clock64();
#endif
  if (l == 0) {  // the serial recursion (cov_step) in one thread's registers; J and cv of
                 // step k+1 load during step k
    double sg[15] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    double nj[9] = {Js[2], Js[3], Js[4], Js[7], Js[8], Js[9], Js[14], Js[18], Js[24]};
    double ncv0 = cvs[0], ncv1 = cvs[1];
    for (int k = 0; k < T; ++k) {
      double j[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) j[e] = nj[e];
      const double cv0 = ncv0, cv1 = ncv1;
      if (k + 1 < T) {
        const double* Jn = Js + 25 * (k + 1);
        nj[0] = Jn[2], nj[1] = Jn[3], nj[2] = Jn[4], nj[3] = Jn[7], nj[4] = Jn[8], nj[5] = Jn[9];
        nj[6] = Jn[14], nj[7] = Jn[18], nj[8] = Jn[24];
        ncv0 = cvs[2 * k + 2], ncv1 = cvs[2 * k + 3];
      }
      cov_step(j, cv0, cv1, sg, Ss + 25 * k);
    }
  }
  __syncthreads();
#ifdef GPM_TCOV_TRACE
  ct[2] = clock64();
#endif
  for (int i = l; i < 25 * T; i += nt) ahcov[i] = Ss[i];
  for (int k = l; k < T; k += nt) {  // tighten_lane_radius (uncertainty.cpp:90-96), parallel in k
    if (t.kind == TASK_AVOIDANCE) break;
    const double r = lane_radius(Ss + 25 * k, t.half_width, a.chi2);
    arbar[k] = r;
    if (r <= 0.0) atomicOr(&infeasible, 1);
  }
  if (t.kind != TASK_TRACKING)  // tighten_obstacle_distance (uncertainty.cpp:98-116), parallel in (k, o)
    for (int idx = l; idx < T * t.n_obs; idx += nt) {
      const int k = idx / t.n_obs, o = idx % t.n_obs;
      const double* mu = mus + (k + 1) * 5;  // belief mean after step k
      double dbar;
      amarg[(size_t)k * t.n_obs + o] = obstacle_margin(Ss + 25 * k, mu[0], mu[1], t.obs[o], a.z, &dbar);
      if (dbar <= 0.0) atomicOr(&infeasible, 1);
    }
  __syncthreads();
  if (l == 0) {
    a.infeasible[rb] = infeasible;
    if (a.done_host) {  // zero-copy: infeasibility, then the tick's sequence number
      const double v = (double)infeasible;
      publish_host(a.done_host + 2 * (size_t)rb, &v, 1, 1, a.x0[(size_t)rb * BatchStrides::X0 + 7]);
    }
  }
#ifdef GPM_TCOV_TRACE
  if (l == 0) printf("tcov: staging+cv %lld recursion %lld thresholds %lld\n", ct[1] - ct[0], ct[2] - ct[1], clock64() - ct[2]);
#endif
  if (threadIdx.x == 0) tl_stamp(12);
}

int tighten_splits(int n, int B) { return n > 0 ? (n + tight_rows(n, B) - 1) / tight_rows(n, B) : 1; }

// Pipelined single-robot covariance pass (a.tflags), launched after the variance grid: it only
// waits on work launched before it (serialisation-safe: under a profiler that runs kernels one
// at a time every flag is already up). Warp 1 stages J_k / mu_k as the mean kernel's publisher
// raises flag 1, warp 2 collects cv_k as the variance grid raises the per-step flags, warp 0
// lane 0 runs the recursion (tighten_cov_kernel's arithmetic) as both arrive, warps 3-7
// evaluate step k's thresholds as soon as Σ_k is known; at the end every flag is lowered.
__global__ void __launch_bounds__(256, 1) tighten_cov_pipe_kernel(const TightenArgs a) {
  pdl_trigger();
  const int T = a.T, l = threadIdx.x, lane = l & 31, w = l >> 5;
  extern __shared__ __align__(16) double psm[];  // [T][9] J, [T][2] cv, [T][25] Σ, [T+1][2] xy, int[T]
  double* const pJ = psm;
  double* const pcv = pJ + 9 * T;
  double* const pS = pcv + 2 * T;
  double* const pxy = pS + 25 * T;
  volatile int* const cv_ready = reinterpret_cast<volatile int*>(pxy + 2 * (T + 1));
  __shared__ volatile int j_ready, mu_ready, s_done;
  __shared__ int infeasible;
  if (l == 0) {
    j_ready = 0;
    mu_ready = 0;
    s_done = 0;
    infeasible = 0;
  }
  for (int i = l; i < T; i += blockDim.x) cv_ready[i] = 0;
  __syncthreads();
  if (w == 1) {  // ---- J / belief-mean stager
    int staged = 0;
    unsigned it = 0;
    while (staged < T + 1) {
      unsigned avail = ld_relaxed_u32(a.tflags + 1);
      avail = __shfl_sync(0xffffffffu, avail, 0);
      if ((int)avail <= staged) {
        __nanosleep(64);
        if (++it > (1u << 25)) {
          printf("tighten_cov_pipe_kernel: Jacobian wait timed out\n");
          __trap();
        }
        continue;
      }
      __threadfence();  // acquire: the rows published before the counter
      const int j0 = staged < T ? staged : T, jt = (int)avail < T ? (int)avail : T;
      for (int i = lane; i < 9 * (jt - j0); i += 32) {  // J = [1 0 a b c; 0 1 d e f; 0 0 1 0 g; 0 0 0 h 0; 0 0 0 0 i]
        const int kk = j0 + i / 9, e = i % 9;
        const int src = e < 3 ? 2 + e : e < 6 ? 4 + e : e == 6 ? 14 : e == 7 ? 18 : 24;
        pJ[kk * 9 + e] = __ldcg(a.tJ + kk * 25 + src);
      }
      for (int i = lane; i < 2 * ((int)avail - staged); i += 32) {
        const int kk = staged + i / 2;
        pxy[2 * kk + (i & 1)] = __ldcg(a.tmu + kk * 5 + (i & 1));
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        j_ready = jt;
        mu_ready = (int)avail;
      }
      staged = (int)avail;
    }
  } else if (w == 2) {  // ---- cv stager: lanes watch a window of 32 steps' flags
    int base = 0;
    unsigned it = 0;
    while (base < T) {
      const int kk = base + lane;
      bool ready = kk >= T;
      if (!ready && !cv_ready[kk] && ld_relaxed_u32(a.tflags + 2 + kk) == 0x40000000u) {
        __threadfence();  // acquire for cv_k
        pcv[2 * kk] = __ldcg(a.tcv + 2 * kk);
        pcv[2 * kk + 1] = __ldcg(a.tcv + 2 * kk + 1);
        __threadfence_block();
        cv_ready[kk] = 1;
      }
      if (!ready) ready = cv_ready[kk] != 0;
      const unsigned all = __ballot_sync(0xffffffffu, ready);
      const int adv = all == 0xffffffffu ? 32 : __ffs(~all) - 1;  // leading run of ready steps
      base += adv;
      if (adv == 0) {
        __nanosleep(64);
        if (++it > (1u << 25)) {
          printf("tighten_cov_pipe_kernel: variance wait timed out\n");
          __trap();
        }
      }
    }
  } else if (w == 0) {  // ---- the covariance recursion (tighten_cov_kernel's), step by step
    if (lane == 0) {
      double sg[15] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int kk = 0; kk < T; ++kk) {
        for (unsigned it = 0; j_ready <= kk || !cv_ready[kk]; ++it) {
          __nanosleep(16);
          if (it > (1u << 27)) __trap();
        }
        __threadfence_block();
        double j[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) j[e] = pJ[9 * kk + e];
        cov_step(j, pcv[2 * kk], pcv[2 * kk + 1], sg, pS + 25 * kk);
        __threadfence_block();
        s_done = kk + 1;
      }
      tl_stamp(24);
    }
    __syncwarp();
  } else {  // ---- warps 3-7: step k's covariance out, lane radius and obstacle margins
    const TaskDev& tk = a.task[0];
    for (int kk = w - 3; kk < T; kk += 5) {
      for (unsigned it = 0; s_done <= kk || mu_ready <= kk + 1; ++it) {
        __nanosleep(32);
        if (it > (1u << 27)) __trap();
      }
      __threadfence_block();
      const double* Sk = pS + 25 * kk;
      if (lane < 25) a.horizon_cov[25 * kk + lane] = Sk[lane];
      if (lane == 0 && tk.kind != TASK_AVOIDANCE) {  // tighten_lane_radius (uncertainty.cpp:90-96)
        const double r = lane_radius(Sk, tk.half_width, a.chi2);
        a.r_bar[kk] = r;
        if (r <= 0.0) atomicOr(&infeasible, 1);
      }
      if (tk.kind != TASK_TRACKING)  // tighten_obstacle_distance (uncertainty.cpp:98-116)
        for (int o = lane; o < tk.n_obs; o += 32) {  // belief mean after step k
          double dbar;
          a.margins[(size_t)kk * tk.n_obs + o] =
              obstacle_margin(Sk, pxy[2 * (kk + 1)], pxy[2 * (kk + 1) + 1], tk.obs[o], a.z, &dbar);
          if (dbar <= 0.0) atomicOr(&infeasible, 1);
        }
    }
  }
  __syncthreads();
  for (int i = l; i < T + 2; i += blockDim.x) a.tflags[i] = 0u;  // every reader of this tick's flags is done
  if (l == 0) {
    a.infeasible[0] = infeasible;
    if (a.done_host) {  // zero-copy: infeasibility, then the tick's sequence number
      const double v = (double)infeasible;
      publish_host(a.done_host, &v, 1, 1, a.x0[7]);
    }
    tl_stamp(12);
  }
}

cudaError_t launch_tighten(const TightenArgs& a, cudaStream_t st) {
  size_t msm = sizeof(double) * (size_t)(2 * a.T + 3 * (a.T + 1) + 2 * a.T + 1);
  if (a.model_kind == MODEL_GP)
    msm += sizeof(double) * (size_t)7 * a.model.ns * a.model.G;  // Z + combined alpha per group
  int no = 1;
  if (a.model_kind == MODEL_GP)
    for (int g = 0; g < a.model.G; ++g) no = a.model.g[g].n_out > no ? a.model.g[g].n_out : no;
  void (*mk)(const TightenArgs) = no <= 2 ? tighten_mean_kernel<2> : no <= 4 ? tighten_mean_kernel<4>
                                  : no <= 6 ? tighten_mean_kernel<6> : tighten_mean_kernel<8>;
  cudaFuncSetAttribute(mk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm);  // static + dynamic may exceed 48 KB
  cudaError_t el = launch_pdl(mk, dim3(a.B), dim3(TMEAN_THREADS + (a.tflags ? 32 : 0)), msm, st, a);
  if (el != cudaSuccess) return el;
  const int G = a.model_kind == MODEL_GP ? a.model.G : 1;
  const int ns = a.model_kind == MODEL_GP ? tighten_splits(a.model.n, a.B) : 1;
  const size_t smem = sizeof(double) * (size_t)(a.model.n > 0 ? a.model.n : 1);
  cudaFuncSetAttribute(tighten_var_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (a.model_kind == MODEL_GP) {
    el = launch_pdl(tighten_var_kernel, dim3(ns, G * a.B, a.T), dim3(256), smem, st, a);
    if (el != cudaSuccess) return el;
  }
  if (a.tflags) {
    const size_t psm = sizeof(double) * (size_t)(9 * a.T + 2 * a.T + 25 * a.T + 2 * (a.T + 1)) + sizeof(int) * a.T;
    cudaFuncSetAttribute(tighten_cov_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
    el = launch_pdl(tighten_cov_pipe_kernel, dim3(1), dim3(256), psm, st, a);
  } else {
    const size_t csmem = sizeof(double) * (size_t)(25 * a.T + 2 * a.T + 5 * (a.T + 1) + 25 * a.T);
    cudaFuncSetAttribute(tighten_cov_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem);
    el = launch_pdl(tighten_cov_kernel, dim3(a.B), dim3(256), csmem, st, a, ns);
  }
  if (el != cudaSuccess) return el;
  count_launch(3);
  return cudaGetLastError();
}

// -------------------------------------------------------------------------
// -------------------------------------------------------------------------
// Reference free functions (mppi.hpp:60-79) as device kernels behind the C ABI.

// mppi.cpp:80-111 rollout(): one block walks the T steps; the GP query of each
// step is the block-wide FP64 predict used by the tightening pass.
__global__ void __launch_bounds__(256) rollout_one_kernel(const ModelDev M, int model_kind, NominalDev nom,
                                                          Edd5Dev edd, const double* x0, const double* seq,
                                                          int T, const double* w, int R, double* states,
                                                          double* corr) {
  extern __shared__ __align__(16) double kst[];
  __shared__ double red[32 * 8];
  __shared__ double smean[kMaxGroups * kMaxOutPerGroup];
  __shared__ double svar[kMaxGroups];
  __shared__ double st[5];
  if (threadIdx.x < 5) {
    st[threadIdx.x] = x0[threadIdx.x];
    states[threadIdx.x] = x0[threadIdx.x];
  }
  __syncthreads();
  for (int k = 0; k < T; ++k) {
    const double u[2] = {seq[2 * k], seq[2 * k + 1]};
    if (model_kind == MODEL_GP) {
      const double q[4] = {st[3], st[4], u[0], u[1]};
      block_gp_predict(M, q, kst, red, smean, svar);
    }
    if (threadIdx.x == 0) {
      double s5[5], nx[5];
      for (int i = 0; i < 5; ++i) s5[i] = st[i];
      double cm0 = 0.0, cm1 = 0.0, vv = 0.0, vw = 0.0;
      if (model_kind == MODEL_GP) {
        double vout[kMaxGroups * kMaxOutPerGroup];
        for (int g = 0; g < M.G; ++g)
          for (int o = 0; o < M.g[g].n_out; ++o) vout[M.g[g].out_idx[o]] = svar[g];
        for (int i = 0; i < R; ++i) {  // combine_terrains, ascending i (mppi.cpp:34-49)
          const double wi = w[i];
          cm0 += wi * smean[2 * i];
          cm1 += wi * smean[2 * i + 1];
          vv += wi * wi * vout[2 * i];
          vw += wi * wi * vout[2 * i + 1];
        }
        double sp, cp;
        sincos(s5[2], &sp, &cp);
        step_nominal(s5, u, nom, nx, sp, cp);
        nx[3] += cm0;
        nx[4] += cm1;
      } else if (model_kind == MODEL_EDD5) {
        step_edd5(s5, u, edd, nom.dt, nx);
      } else if (model_kind == MODEL_UNICYCLE) {
        step_kinematic(s5, u, nom.dt, nx);
      } else {
        double sp, cp;
        sincos(s5[2], &sp, &cp);
        step_nominal(s5, u, nom, nx, sp, cp);
      }
      for (int i = 0; i < 5; ++i) {
        st[i] = nx[i];
        states[5 * (k + 1) + i] = nx[i];
      }
      corr[4 * k] = cm0;
      corr[4 * k + 1] = cm1;
      corr[4 * k + 2] = vv;
      corr[4 * k + 3] = vw;
    }
    __syncthreads();
  }
}

cudaError_t launch_rollout_one(const ModelDev& M, int model_kind, const NominalDev& nom, const Edd5Dev& edd,
                               const double* x0, const double* seq, int T, const double* w, int R,
                               double* states, double* corr, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)(model_kind == MODEL_GP ? M.n : 1);
  cudaError_t e = cudaFuncSetAttribute(rollout_one_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  rollout_one_kernel<<<1, 256, smem, st>>>(M, model_kind, nom, edd, x0, seq, T, w, R, states, corr);
  count_launch();
  return cudaGetLastError();
}

// mppi.cpp:125-145 trajectory_weights: one block (block min, exp, sum, scale).
__global__ void __launch_bounds__(1024) trajectory_weights_kernel(const double* c, long long K, double lambda,
                                                                  double* w) {
  __shared__ double red[32 * 5];
  double lmin = INFINITY;
  for (long long i = threadIdx.x; i < K; i += blockDim.x)
    if (isfinite(c[i])) lmin = fmin(lmin, c[i]);
  lmin = warp_min(lmin);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lmin;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = INFINITY;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmin(m, red[i]);
    red[31 * 5] = m;
  }
  __syncthreads();
  const double m = red[31 * 5];
  __syncthreads();
  if (!isfinite(m)) {  // no valid sample this tick: all zeros
    for (long long i = threadIdx.x; i < K; i += blockDim.x) w[i] = 0.0;
    return;
  }
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (long long i = threadIdx.x; i < K; i += blockDim.x) {
    const double e = isfinite(c[i]) ? exp(-(c[i] - m) / lambda) : 0.0;
    w[i] = e;
    v[0] += e;
  }
  block_reduce_5(v, red);
  const double Z = v[0];
  for (long long i = threadIdx.x; i < K; i += blockDim.x) w[i] = w[i] / Z;
}

// mppi.cpp:147-164 update_controls: thread per (k, component), samples in index order.
__global__ void update_controls_kernel(const double* nom, int T, const double* eps, const double* w, long long K,
                                       double lo0, double lo1, double hi0, double hi1, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * T) return;
  const int k = i >> 1, c = i & 1;
  double d = 0.0;
  for (long long s = 0; s < K; ++s) d += w[s] * eps[((size_t)s * T + k) * 2 + c];
  out[i] = clampd(nom[i] + d, c ? lo1 : lo0, c ? hi1 : hi0);
}

// mppi.cpp:166-173 shift_horizon
__global__ void shift_horizon_kernel(const double* seq, int T, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * T) return;
  const int k = i >> 1;
  out[i] = seq[2 * (k + 1 < T ? k + 1 : T - 1) + (i & 1)];
}

cudaError_t launch_trajectory_weights(const double* c, long long K, double lambda, double* w, cudaStream_t st) {
  trajectory_weights_kernel<<<1, 1024, 0, st>>>(c, K, lambda, w);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_update_controls(const double* nom, int T, const double* eps, const double* w, long long K,
                                   const double lo[2], const double hi[2], double* out, cudaStream_t st) {
  update_controls_kernel<<<(2 * T + 127) / 128, 128, 0, st>>>(nom, T, eps, w, K, lo[0], lo[1], hi[0], hi[1], out);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_shift_horizon(const double* seq, int T, double* out, cudaStream_t st) {
  shift_horizon_kernel<<<(2 * T + 127) / 128, 128, 0, st>>>(seq, T, out);
  count_launch();
  return cudaGetLastError();
}

__global__ void philox_noise_kernel(uint64_t key, long long s_begin, int K, int T, double sv,
                                    double sw, double* eps) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)K * T) return;
  const long long s = i / T;
  const int k = (int)(i % T);
  double z1, z2;
  philox_gaussian_pair(key, (uint64_t)(s_begin + s), (uint32_t)k, &z1, &z2);
  eps[2 * i] = sv * z1;
  eps[2 * i + 1] = sw * z2;
}

cudaError_t launch_philox_noise(uint64_t key, long long s_begin, int K, int T, double sv,
                                double sw, double* eps, cudaStream_t st) {
  const long long n = (long long)K * T;
  philox_noise_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(key, s_begin, K, T, sv, sw, eps);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gpm
