// capi.cpp — C++ host layer behind include/gpmppi_b200.h.
//
// Owns the GP model (host FP64 factorisation restating gp.cpp:61-150, device
// upload) and the planner (device buffers, stream, per-tick orchestration of
// the kernels in kernels.cu, restating Planner::plan_step_impl, mppi.cpp:389-462).
#include "gpmppi_b200.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "internal.hpp"

namespace {

// NVTX ranges (header-only NVTX3: free when no tool is attached) around the host phases of
// a tick and the enqueue of each device phase, for nsys / ncu --nvtx.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct CudaError {
  cudaError_t e;
  const char* where;
};

#define CK(call)                                                          \
  do {                                                                    \
    cudaError_t e__ = (call);                                             \
    if (e__ != cudaSuccess) throw CudaError{e__, #call};                  \
  } while (0)

struct NcclError {
  std::string msg;
};

struct ArgError {
  int code;
  std::string msg;
};
[[noreturn]] void invalid(const std::string& m) { throw ArgError{GPMPPI_INVALID_ARGUMENT, m}; }
[[noreturn]] void runtime(const std::string& m) { throw ArgError{GPMPPI_RUNTIME_ERROR, m}; }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return GPMPPI_OK;
  } catch (const ArgError& e) {
    return fail(e.code, e.msg);
  } catch (const CudaError& e) {
    return fail(GPMPPI_CUDA_ERROR, std::string("CUDA error in ") + e.where + ": " +
                                       cudaGetErrorString(e.e));
  } catch (const NcclError& e) {
    return fail(GPMPPI_RUNTIME_ERROR, e.msg);
  } catch (const std::bad_alloc&) {
    return fail(GPMPPI_RUNTIME_ERROR, "host allocation failed");
  }
}

void require_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw CudaError{e == cudaSuccess ? cudaErrorNoDevice : e, "cudaGetDeviceCount (no CUDA device)"};
  if (device < 0 || device >= count) invalid("device index out of range");
  CK(cudaSetDevice(device));
}

// ---------------------------------------------------------------------------
// NCCL, resolved at run time from the libnccl.so.2 the process already has (torch's) or
// the system one: the sharded solve's one collective (mppi.cpp:428-429 is the reference's
// only exchange point) runs on the planner stream inside the library.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};
const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.comm_destroy) a.why = "libnccl lacks a symbol";
    return a;
  }();
  return api;
}
void nccl_check(ncclResult_t r, const char* where) {
  if (r != ncclSuccess) {
    const NcclApi& a = nccl_api();
    throw NcclError{std::string("NCCL error in ") + where + ": " +
                    (a.error_string ? a.error_string(r) : std::to_string((int)r))};
  }
}
const NcclApi& nccl_required() {
  const NcclApi& a = nccl_api();
  if (!a.why.empty()) throw NcclError{a.why};
  return a;
}

// ---------------------------------------------------------------------------
// Host FP64 GP factorisation (gp.cpp:61-150).
struct HostGroup {
  double kernel[6];
  std::vector<int> outputs;
  double jitter = 0.0;
  std::vector<double> aug;    // n×6 [x/l | 1 | -1/2|x/l|^2 + ln sv]  (gp.cpp:103-110)
  std::vector<double> chol;   // n×n lower
  std::vector<double> ilt;    // n×n upper = L^{-T}
  std::vector<double> alphas; // n×n_out
};

bool cholesky_lower(std::vector<double>& A, int n) {  // Eigen LLT: fail iff a pivot <= 0
  for (int j = 0; j < n; ++j) {
    double* rj = &A[(size_t)j * n];
    double x = rj[j];
    for (int k = 0; k < j; ++k) x -= rj[k] * rj[k];
    if (!(x > 0.0)) return false;
    const double d = std::sqrt(x);
    rj[j] = d;
    for (int i = j + 1; i < n; ++i) {
      double* ri = &A[(size_t)i * n];
      double v = ri[j];
      for (int k = 0; k < j; ++k) v -= ri[k] * rj[k];
      ri[j] = v / d;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A[(size_t)i * n + j] = 0.0;
  return true;
}

// Device factorisation (fit.cu) for n >= 1024, where the O(n^3) host loops take
// seconds; GPMPPI_FIT=host|device overrides.
bool device_fit(int n) {
  const char* e = std::getenv("GPMPPI_FIT");
  if (e && std::strcmp(e, "host") == 0) return false;
  if (e && std::strcmp(e, "device") == 0) return true;
  return n >= 1024;
}

void factor_group(HostGroup& G, const double* X, const double* Y, int n, int m,
                  std::vector<double>& lml) {
  const double sv = G.kernel[0], nv = G.kernel[5];
  G.aug.assign((size_t)n * 6, 0.0);
  std::vector<double> norms(n);
  for (int i = 0; i < n; ++i) {
    double sq = 0.0;
    for (int d = 0; d < 4; ++d) {
      const double v = X[(size_t)i * 4 + d] / G.kernel[1 + d];
      G.aug[(size_t)i * 6 + d] = v;
      sq += v * v;
    }
    norms[i] = -0.5 * sq;
    G.aug[(size_t)i * 6 + 4] = 1.0;
    G.aug[(size_t)i * 6 + 5] = norms[i] + std::log(sv);
  }
  std::vector<double> K((size_t)n * n);  // gp.cpp:112-114
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double* a = &G.aug[(size_t)i * 6];
      const double* b = &G.aug[(size_t)j * 6];
      K[(size_t)i * n + j] = std::exp(a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3] +
                                      norms[i] + b[5]);
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double s = 0.5 * (K[(size_t)i * n + j] + K[(size_t)j * n + i]);
      K[(size_t)i * n + j] = K[(size_t)j * n + i] = s;
    }
  std::vector<double> Xi;  // L^{-1}, row-major lower
  if (device_fit(n)) {  // gp.cpp:116-138 on the device (fit.cu)
    bool ok = false;
    double jitter = 0.0;
    G.chol.assign((size_t)n * n, 0.0);
    Xi.assign((size_t)n * n, 0.0);
    CK(gpm::device_factor(K.data(), n, nv, G.chol.data(), Xi.data(), &jitter, &ok));
    if (!ok) {
      std::ostringstream msg;
      msg << "GpModel::fit: Cholesky failed for kernel group after jitter up to 1e-6"
          << " (signal_var=" << sv << ", noise_var=" << nv << ")";
      runtime(msg.str());
    }
    G.jitter = jitter;
  } else {
    bool ok = false;  // gp.cpp:116-133 jitter ladder
    double jitter = 0.0;
    for (int attempt = 0; attempt <= 5 && !ok; ++attempt) {
      jitter = attempt == 0 ? 0.0 : std::pow(10.0, -11 + attempt);
      G.chol = K;
      for (int i = 0; i < n; ++i) G.chol[(size_t)i * n + i] += nv + jitter;
      ok = cholesky_lower(G.chol, n);
    }
    if (!ok) {
      std::ostringstream msg;
      msg << "GpModel::fit: Cholesky failed for kernel group after jitter up to 1e-6"
          << " (signal_var=" << sv << ", noise_var=" << nv << ")";
      runtime(msg.str());
    }
    G.jitter = jitter;
    const std::vector<double>& Lh = G.chol;
    // L^{-1} row by row (axpy form), then transpose (gp.cpp:135-138)
    Xi.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) {
      double* xi = &Xi[(size_t)i * n];
      xi[i] = 1.0;
      for (int k = 0; k < i; ++k) {
        const double l = Lh[(size_t)i * n + k];
        const double* xk = &Xi[(size_t)k * n];
        for (int c = 0; c <= k; ++c) xi[c] -= l * xk[c];
      }
      const double d = Lh[(size_t)i * n + i];
      for (int c = 0; c <= i; ++c) xi[c] /= d;
    }
  }
  const std::vector<double>& L = G.chol;
  G.ilt.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = i; j < n; ++j) G.ilt[(size_t)i * n + j] = Xi[(size_t)j * n + i];
  // alphas + LML (gp.cpp:140-147)
  const int no = (int)G.outputs.size();
  G.alphas.assign((size_t)n * no, 0.0);
  double logdet = 0.0;
  for (int i = 0; i < n; ++i) logdet += std::log(L[(size_t)i * n + i]);
  std::vector<double> z(n);
  const double log2pi = std::log(2.0 * gpm::kPi);
  for (int c = 0; c < no; ++c) {
    const int j = G.outputs[c];
    for (int i = 0; i < n; ++i) {
      double v = Y[(size_t)i * m + j];
      const double* li = &L[(size_t)i * n];
      for (int k = 0; k < i; ++k) v -= li[k] * z[k];
      z[i] = v / li[i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double v = z[i];
      for (int k = i + 1; k < n; ++k) v -= L[(size_t)k * n + i] * G.alphas[(size_t)k * no + c];
      G.alphas[(size_t)i * no + c] = v / L[(size_t)i * n + i];
    }
    double dot = 0.0;
    for (int i = 0; i < n; ++i) dot += Y[(size_t)i * m + j] * G.alphas[(size_t)i * no + c];
    lml[j] = -0.5 * dot - logdet - 0.5 * (double)n * log2pi;
  }
}

}  // namespace

namespace gpm_host {  // error channel for the other translation units (hostapi.cpp)
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace gpm_host

// ===========================================================================
struct gpmppi_model {
  int device = 0;
  int n = 0, m = 0;
  std::vector<double> inputs, outputs, kernels, lml;
  std::vector<HostGroup> groups;
  std::vector<void*> dev_allocs;
  gpm::ModelDev dev{};
  ~gpmppi_model() {
    cudaSetDevice(device);
    for (void* p : dev_allocs) cudaFree(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(v.size(), 1)));
    dev_allocs.push_back(p);
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return static_cast<T*>(p);
  }
};

namespace {

gpmppi_model* build_model(const double* X, const double* Y, int64_t n64, int64_t m64,
                          const double* kernels, int device) {
  if (n64 < 1) invalid("GpModel::fit: inputs must be n x 4 with n >= 1");
  if (m64 < 1) invalid("GpModel::fit: outputs must be n x m with m >= 1");
  if (n64 > (1 << 16)) invalid("GpModel::fit: n too large for the device model");
  const int n = (int)n64, m = (int)m64;
  for (size_t i = 0; i < (size_t)n * 4; ++i)
    if (!std::isfinite(X[i])) invalid("GpModel::fit: non-finite training data");
  for (size_t i = 0; i < (size_t)n * m; ++i)
    if (!std::isfinite(Y[i])) invalid("GpModel::fit: non-finite training data");
  std::vector<HostGroup> groups;
  for (int j = 0; j < m; ++j) {  // gp.cpp:85-100
    const double* kp = kernels + 6 * j;
    bool ok = kp[0] > 0.0 && kp[5] > 0.0;
    for (int d = 0; d < 4; ++d) ok = ok && kp[1 + d] > 0.0;
    if (!ok) invalid("KernelParams: all parameters must be strictly positive");
    int g = -1;
    for (size_t k = 0; k < groups.size(); ++k)
      if (std::memcmp(groups[k].kernel, kp, sizeof(double) * 6) == 0) g = (int)k;
    if (g < 0) {
      groups.emplace_back();
      std::memcpy(groups.back().kernel, kp, sizeof(double) * 6);
      g = (int)groups.size() - 1;
    }
    groups[g].outputs.push_back(j);
  }
  if ((int)groups.size() > gpm::kMaxGroups)
    invalid("GpModel::fit: at most " + std::to_string(gpm::kMaxGroups) + " distinct kernels supported on device");
  for (auto& g : groups)
    if ((int)g.outputs.size() > gpm::kMaxOutPerGroup)
      invalid("GpModel::fit: at most " + std::to_string(gpm::kMaxOutPerGroup) + " outputs per kernel supported on device");
  require_device(device);
  auto* M = new gpmppi_model();
  try {
    M->device = device;
    M->n = n;
    M->m = m;
    M->inputs.assign(X, X + (size_t)n * 4);
    M->outputs.assign(Y, Y + (size_t)n * m);
    M->kernels.assign(kernels, kernels + (size_t)m * 6);
    M->lml.assign(m, 0.0);
    M->groups = std::move(groups);
    for (auto& G : M->groups) factor_group(G, X, Y, n, m, M->lml);
    // device upload
    M->dev.n = n;
    M->dev.m = m;
    M->dev.G = (int)M->groups.size();
    M->dev.ns = (n + 1) & ~1;
    M->dev.fold_zn = 1;
    for (const HostGroup& G : M->groups) {
      if (!(std::fabs(std::log(G.kernel[0])) <= 50.0)) M->dev.fold_zn = 0;
      for (int j = 0; j < n; ++j)
        if (!(std::fabs(G.aug[(size_t)j * 6 + 5]) <= 600.0)) M->dev.fold_zn = 0;
    }
    if (const char* e = getenv("GPMPPI_FOLD_ZN")) M->dev.fold_zn = M->dev.fold_zn && atoi(e) != 0;
    for (int gi = 0; gi < M->dev.G; ++gi) {
      const HostGroup& G = M->groups[gi];
      gpm::GroupDev& D = M->dev.g[gi];
      const int no = (int)G.outputs.size();
      const int ns = M->dev.ns;
      std::vector<double> pts((size_t)(5 + no) * ns, 0.0);
      for (int j = 0; j < ns; ++j) {
        if (j >= n) {  // padding point: k* = exp(-1e300) = 0, alpha = 0
          pts[(size_t)4 * ns + j] = -1e300;
          continue;
        }
        for (int d = 0; d < 4; ++d) pts[(size_t)d * ns + j] = G.aug[(size_t)j * 6 + d];
        pts[(size_t)4 * ns + j] = G.aug[(size_t)j * 6 + 5];
        for (int c = 0; c < no; ++c) pts[(size_t)(5 + c) * ns + j] = G.alphas[(size_t)j * no + c];
      }
      std::vector<float> ilt32(G.ilt.size()), zs32((size_t)4 * n);
      for (size_t i = 0; i < G.ilt.size(); ++i) ilt32[i] = (float)G.ilt[i];
      for (int j = 0; j < n; ++j)
        for (int d = 0; d < 4; ++d) zs32[(size_t)d * n + j] = (float)G.aug[(size_t)j * 6 + d];
      D.pts = M->upload(pts);
      D.ilt64 = M->upload(G.ilt);
      {  // L^{-1} row-major: the tightening variance reads row j contiguously (coalesced)
        std::vector<double> linv((size_t)n * n);
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) linv[(size_t)j * n + i] = G.ilt[(size_t)i * n + j];
        D.linv64 = M->upload(linv);
      }
      D.ilt32 = M->upload(ilt32);
      D.zs32 = M->upload(zs32);
      {  // tensor-core operand (pre-tiled TF32 hi/lo L^{-T}, kernels_tc.cu)
        std::vector<float> tcd;
        std::vector<int4> tcm;
        gpm::build_tc_operand(G.ilt.data(), n, tcd, tcm, D.tc_npad, D.tc_np, D.tc_npass);
        D.tc_b = M->upload(tcd);
        D.tc_meta = M->upload(tcm);
        std::vector<uint16_t> tch;
        std::vector<int4> tchm;
        gpm::build_tc_operand_f16(G.ilt.data(), n, G.kernel[0], D.tc_npad, D.tc_np, D.tc_npass, tch, tchm, D.tc_hfac);
        D.tc_h = M->upload(tch);
        D.tc_hmeta = M->upload(tchm);
        gpm::build_tc_operand_f16x2(G.ilt.data(), n, G.kernel[0], D.tc_npad, tch, tchm, D.tc_npass2);
        D.tc_h2 = M->upload(tch);
        D.tc_h2meta = M->upload(tchm);
      }
      for (int d = 0; d < 4; ++d) D.ls[d] = G.kernel[1 + d];
      D.sv = G.kernel[0];
      D.log_sv = std::log(G.kernel[0]);
      D.n_out = no;
      for (int c = 0; c < gpm::kMaxOutPerGroup; ++c) D.out_idx[c] = c < no ? G.outputs[c] : 0;
    }
  } catch (...) {
    delete M;
    throw;
  }
  return M;
}

const char kGpMagic[8] = {'G', 'P', 'M', 'P', 'P', 'I', 'G', '1'};      // gp.cpp:19
const char kModelsMagic[8] = {'G', 'P', 'M', 'P', 'P', 'I', 'M', '1'};  // harness.cpp:19

// GpModel::load(std::istream&) (gp.cpp:250-272): column-major f64 records, refit.
gpmppi_model* load_gp_stream(std::istream& is, int device) {
  auto read_raw = [&](void* p, size_t bytes) {
    is.read(static_cast<char*>(p), (std::streamsize)bytes);
    if (!is) runtime("GpModel::load: truncated record");
  };
  char magic[8];
  read_raw(magic, 8);
  if (std::memcmp(magic, kGpMagic, 8) != 0) runtime("GpModel::load: bad magic");
  int64_t n = 0, m = 0;
  read_raw(&n, 8);
  read_raw(&m, 8);
  if (n < 1 || m < 1 || n > (1 << 24) || m > (1 << 16)) runtime("GpModel::load: implausible dimensions");
  std::vector<double> cin((size_t)n * 4), cout((size_t)n * m), kern((size_t)m * 6);
  read_raw(cin.data(), sizeof(double) * cin.size());
  read_raw(cout.data(), sizeof(double) * cout.size());
  read_raw(kern.data(), sizeof(double) * kern.size());  // per output: sv, l0..l3, nv
  std::vector<double> X((size_t)n * 4), Y((size_t)n * m);  // column-major -> row-major
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 4; ++d) X[(size_t)i * 4 + d] = cin[(size_t)d * n + i];
    for (int64_t j = 0; j < m; ++j) Y[(size_t)i * m + j] = cout[(size_t)j * n + i];
  }
  return build_model(X.data(), Y.data(), n, m, kern.data(), device);
}

// GpModel::save(std::ostream&) (gp.cpp:230-242)
void save_gp_stream(std::ostream& os, const gpmppi_model* M) {
  const int64_t n = M->n, m = M->m;
  os.write(kGpMagic, 8);
  os.write(reinterpret_cast<const char*>(&n), 8);
  os.write(reinterpret_cast<const char*>(&m), 8);
  std::vector<double> cin((size_t)n * 4), cout((size_t)n * m);
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 4; ++d) cin[(size_t)d * n + i] = M->inputs[(size_t)i * 4 + d];
    for (int64_t j = 0; j < m; ++j) cout[(size_t)j * n + i] = M->outputs[(size_t)i * m + j];
  }
  os.write(reinterpret_cast<const char*>(cin.data()), sizeof(double) * cin.size());
  os.write(reinterpret_cast<const char*>(cout.data()), sizeof(double) * cout.size());
  os.write(reinterpret_cast<const char*>(M->kernels.data()), sizeof(double) * M->kernels.size());
}

}  // namespace

extern "C" {

const char* gpmppi_last_error(void) { return g_err.c_str(); }
int gpmppi_abi_version(void) { return GPMPPI_ABI_VERSION; }
uint64_t gpmppi_kernel_launches(void) { return gpm::launches_total(); }

int gpmppi_model_fit(const double* inputs, const double* outputs, int64_t n, int64_t m,
                     const double* kernels, int device, gpmppi_model** out) {
  if (!out) return fail(GPMPPI_INVALID_ARGUMENT, "null output handle");
  *out = nullptr;
  return guarded([&] { *out = build_model(inputs, outputs, n, m, kernels, device); });
}

int gpmppi_model_load(const char* path, int device, gpmppi_model** out) {  // gp.cpp:244-248
  if (!out) return fail(GPMPPI_INVALID_ARGUMENT, "null output handle");
  *out = nullptr;
  return guarded([&] {
    std::ifstream is(path ? path : "", std::ios::binary);
    if (!is) runtime(std::string("GpModel::load: cannot open ") + (path ? path : ""));
    *out = load_gp_stream(is, device);
  });
}

int gpmppi_model_save(const gpmppi_model* M, const char* path) {  // gp.cpp:223-228
  if (!M) return fail(GPMPPI_INVALID_ARGUMENT, "null model");
  return guarded([&] {
    std::ofstream os(path ? path : "", std::ios::binary);
    if (!os) runtime(std::string("GpModel::save: cannot open ") + (path ? path : ""));
    save_gp_stream(os, M);
    if (!os) runtime(std::string("GpModel::save: write failed for ") + path);
  });
}

int gpmppi_models_load(const char* path, int device, gpmppi_edd5* edd5, gpmppi_nominal* nominal,
                       gpmppi_model** gp) {  // harness.cpp:264-284
  if (!gp) return fail(GPMPPI_INVALID_ARGUMENT, "null output handle");
  *gp = nullptr;
  return guarded([&] {
    std::ifstream is(path ? path : "", std::ios::binary);
    if (!is) runtime(std::string("load_models: cannot open ") + (path ? path : ""));
    char magic[8];
    is.read(magic, 8);
    if (!is || std::memcmp(magic, kModelsMagic, 8) != 0)
      runtime(std::string("load_models: bad magic in ") + (path ? path : ""));
    double e[5], nm[3];
    char has_gp = 0;
    is.read(reinterpret_cast<char*>(e), sizeof e);
    is.read(reinterpret_cast<char*>(nm), sizeof nm);
    is.read(&has_gp, 1);
    if (!is) runtime(std::string("load_models: truncated file ") + (path ? path : ""));
    if (edd5) *edd5 = {e[0], e[1], e[2], e[3], e[4]};
    if (nominal) *nominal = {nm[0], nm[1], nm[2]};
    if (has_gp) *gp = load_gp_stream(is, device);
  });
}

int gpmppi_models_save(const char* path, const gpmppi_edd5* edd5, const gpmppi_nominal* nominal,
                       const gpmppi_model* gp) {  // harness.cpp:249-262
  if (!edd5 || !nominal) return fail(GPMPPI_INVALID_ARGUMENT, "save_models: null argument");
  return guarded([&] {
    std::ofstream os(path ? path : "", std::ios::binary);
    if (!os) runtime(std::string("save_models: cannot open ") + (path ? path : ""));
    os.write(kModelsMagic, 8);
    const double e[5] = {edd5->alpha_l, edd5->alpha_r, edd5->x_icr, edd5->y_icr_l, edd5->y_icr_r};
    const double nm[3] = {nominal->tau_v, nominal->tau_omega, nominal->dt};
    os.write(reinterpret_cast<const char*>(e), sizeof e);
    os.write(reinterpret_cast<const char*>(nm), sizeof nm);
    const char has_gp = gp ? 1 : 0;
    os.write(&has_gp, 1);
    if (gp) save_gp_stream(os, gp);
    if (!os) runtime(std::string("save_models: write failed for ") + path);
  });
}

void gpmppi_model_free(gpmppi_model* M) { delete M; }
int gpmppi_model_n_points(const gpmppi_model* M) { return M ? M->n : 0; }
int gpmppi_model_n_outputs(const gpmppi_model* M) { return M ? M->m : 0; }
int gpmppi_model_n_groups(const gpmppi_model* M) { return M ? (int)M->groups.size() : 0; }
double gpmppi_model_group_jitter(const gpmppi_model* M, int g) {
  return (M && g >= 0 && g < (int)M->groups.size()) ? M->groups[g].jitter : NAN;
}
double gpmppi_model_log_marginal_likelihood(const gpmppi_model* M, int o) {
  return (M && o >= 0 && o < M->m) ? M->lml[o] : NAN;
}
int gpmppi_model_training_data(const gpmppi_model* M, double* inputs, double* outputs) {
  if (!M) return fail(GPMPPI_INVALID_ARGUMENT, "null model");
  if (inputs) std::memcpy(inputs, M->inputs.data(), sizeof(double) * M->inputs.size());
  if (outputs) std::memcpy(outputs, M->outputs.data(), sizeof(double) * M->outputs.size());
  return GPMPPI_OK;
}

int gpmppi_model_predict_batch(const gpmppi_model* M, const double* q, int64_t S, double* mean,
                               double* var) {  // gp.cpp:152-207
  if (!M) return fail(GPMPPI_LOGIC_ERROR, "GpModel::predict_batch: model not fitted");
  if (S < 0) return fail(GPMPPI_INVALID_ARGUMENT, "GpModel::predict_batch: queries must be S x 4");
  if (S == 0) return GPMPPI_OK;
  for (int64_t i = 0; i < S * 4; ++i)
    if (!std::isfinite(q[i])) return fail(GPMPPI_INVALID_ARGUMENT, "GpModel::predict: non-finite query");
  return guarded([&] {
    CK(cudaSetDevice(M->device));
    double *dq = nullptr, *dm = nullptr, *dv = nullptr;
    CK(cudaMalloc(&dq, sizeof(double) * S * 4));
    CK(cudaMalloc(&dm, sizeof(double) * S * M->m));
    CK(cudaMalloc(&dv, sizeof(double) * S * M->m));
    CK(cudaMemcpy(dq, q, sizeof(double) * S * 4, cudaMemcpyHostToDevice));
    cudaError_t e = gpm::launch_predict(M->dev, dq, S, dm, dv, 0);
    if (e == cudaSuccess) e = cudaMemcpy(mean, dm, sizeof(double) * S * M->m, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(var, dv, sizeof(double) * S * M->m, cudaMemcpyDeviceToHost);
    cudaFree(dq);
    cudaFree(dm);
    cudaFree(dv);
    if (e != cudaSuccess) throw CudaError{e, "predict_kernel"};
  });
}

int gpmppi_model_variance_batch(const gpmppi_model* M, const double* q, int64_t S, int path,
                                double* var) {
  if (!M) return fail(GPMPPI_LOGIC_ERROR, "GpModel::predict_batch: model not fitted");
  if (S < 0 || path < 0 || path > 4) return fail(GPMPPI_INVALID_ARGUMENT, "variance_batch: bad arguments");
  if (S == 0) return GPMPPI_OK;
  return guarded([&] {
    CK(cudaSetDevice(M->device));
    std::vector<float4> qf(S);
    for (int64_t i = 0; i < S; ++i)
      qf[i] = make_float4((float)q[i * 4], (float)q[i * 4 + 1], (float)q[i * 4 + 2], (float)q[i * 4 + 3]);
    float4* dq = nullptr;
    double* dv = nullptr;
    CK(cudaMalloc(&dq, sizeof(float4) * S));
    CK(cudaMalloc(&dv, sizeof(double) * S));
    cudaError_t e = cudaMemcpy(dq, qf.data(), sizeof(float4) * S, cudaMemcpyHostToDevice);
    std::vector<double> hv(S);
    for (int g = 0; g < M->dev.G && e == cudaSuccess; ++g) {
      gpm::VarianceArgs v{};
      v.queries = dq;
      v.KT = S;
      v.n = M->n;
      v.g = M->dev.g[g];
      v.coef = 1.0;
      v.accumulate = 0;
      v.trace = dv;
      e = gpm::launch_variance(v, path, 0);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e == cudaSuccess) e = cudaMemcpy(hv.data(), dv, sizeof(double) * S, cudaMemcpyDeviceToHost);
      for (int64_t i = 0; i < S && e == cudaSuccess; ++i) var[i * M->dev.G + g] = hv[i];
    }
    cudaFree(dq);
    cudaFree(dv);
    if (e != cudaSuccess) throw CudaError{e, "variance kernel"};
  });
}

}  // extern "C"

// ===========================================================================
struct gpmppi_planner {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;                   // command readback branch (concurrent with tightening)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  int num_sms = 148;
  gpmppi_mppi_config cfg{};
  int model_kind = 0;
  const gpmppi_model* model = nullptr;
  int R = 1;
  int B = 1;                    // robots (independent planners sharing the model)
  std::vector<uint64_t> seeds;  // [B] noise seed of each robot
  gpm::Edd5Dev edd5{};
  gpm::NominalDev nom{};
  double p_x = 0.95, chi2 = 0.0, z = 0.0;
  std::vector<double> tw;  // [B][R]
  uint64_t tick = 0;
  int noise_mode = gpm::NOISE_PHILOX;
  bool injected_set = false;
  int var_path = GPMPPI_VAR_TC_3XF16;  // tensor cores within the stated tolerance
  long long s_begin = 0, K_local = 0, K_total = 0;
  std::vector<uint8_t> rbar_init;  // [B]
  std::vector<int> margins_O;      // [B] obstacle count the margins were sized for
  int n_obs_max = 0;
  int reduce_blocks = 1;  // per robot
  int T = 0, words = 1;
  // device buffers (robot-major, strides in gpm::BatchStrides)
  std::vector<void*> allocs;
  double *d_nom = nullptr, *d_tw = nullptr, *d_x0 = nullptr, *d_rbar = nullptr, *d_margins = nullptr;
  double* d_eps = nullptr;
  double* d_noise = nullptr;  // Philox noise drawn by the rollout, read back by the reduce [B][K][T][2]
  gpm::RolloutGeom geom{};    // GP rollout geometry (query layout), fixed per sample-buffer set
  long long q_slots = 0;      // item-major query / trace slots (gpm::query_slots)
  unsigned long long* d_progress = nullptr;  // per lane group: query steps published (concurrent variance)
  long long progress_words = 0;
  bool coop_ok = false;  // the variance runs concurrently with the rollout (variance_coop_kernel)
  int coop_budget = 0;   // rollout block shared-memory cap that leaves room for it
  gpm::TaskDev* d_task = nullptr;
  double *d_cost_mean = nullptr, *d_var = nullptr, *d_costs = nullptr, *d_e = nullptr;
  float4* d_queries = nullptr;
  uint32_t *d_viol = nullptr, *d_coll = nullptr;
  uint8_t *d_term = nullptr, *d_alive = nullptr;
  double *d_partials = nullptr, *d_rank_tuple = nullptr, *d_out = nullptr, *d_hcov = nullptr,
         *d_combined = nullptr;
  unsigned int* d_ticket = nullptr;
  int* d_infeasible = nullptr;
  double *d_tq = nullptr, *d_tmu = nullptr, *d_tJ = nullptr, *d_tvar = nullptr;
  unsigned int* d_tflags = nullptr;  // pipelined single-robot tightening (TightenArgs::tflags)
  double* d_tcv = nullptr;            // its per-step combined correction variances
  double* d_scratch = nullptr;
  // pinned staging
  gpm::TaskDev* h_task = nullptr;  // [B] (inside the h_x0 block)
  double* h_x0 = nullptr;          // [B][8] robot tick blocks, then the tasks
  const double* dh_x0 = nullptr;   // its mapped device address (stage_tick_kernel), null: copy node
  size_t tick_bytes = 0;
  double* h_out = nullptr;         // [B][16], mapped: the reduce writes command + diag + sequence here
  int* h_infeasible = nullptr;     // [B]
  double* h_done = nullptr;        // [B][2], mapped: tightening infeasibility + sequence
  double *d_out_host = nullptr, *d_done_host = nullptr;  // their device addresses
  // zero-copy completion (default; GPMPPI_ZEROCOPY=0 restores the D2H copies + events): the
  // kernels publish the command and the tightening result into mapped pinned memory behind a
  // per-tick sequence number that plan_step polls
  bool zero_copy = !(getenv("GPMPPI_ZEROCOPY") && atoi(getenv("GPMPPI_ZEROCOPY")) == 0);
  bool zc_tick = false;   // set while the plan_step tick is enqueued / captured
  double seq = 0.0;       // sequence number of the tick being planned
  cudaEvent_t ev[8] = {};
  // one CUDA graph per tick configuration: H2D staging, the six kernels, the command
  // and diagnostics D2H (GPMPPI_NO_GRAPH=1 launches them one by one instead)
  cudaGraph_t tick_graph = nullptr;
  cudaGraphExec_t tick_exec = nullptr;
  long long graph_key = -1;
  int graph_launches = 0;
  bool use_graph = getenv("GPMPPI_NO_GRAPH") == nullptr;
  // sharded solve over NCCL (gpmppi_planner_attach_comm): this rank rolls out its global
  // sample range, the (2T+6)-double tuples are all-gathered on `stream`, every rank combines
  ncclComm_t comm = nullptr;
  int n_ranks = 1, rank = 0;
  double* d_gathered = nullptr;  // [n_ranks][W]
  // command-first mode: plan_step returns once the command is on the host; the tightening
  // pass (consumed only by the next tick, mppi.cpp:235-248) completes behind it
  bool command_first = false;
  bool tightening_pending = false;
  double pending_cmd_ms = 0.0;
  std::chrono::steady_clock::time_point pending_t0;
  std::vector<gpmppi_diag> pending_diag;  // [B], completed by wait_tightening

  std::vector<void*> sample_allocs;  // per-sample buffers, reallocated by set_shard
  static constexpr long long kNoiseMatMax = 1LL << 31;  // sample-steps (config-5 sweep: materialise always)
  template <class T>
  T* dalloc(size_t count, std::vector<void*>* owner = nullptr) {
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
    (owner ? owner : &allocs)->push_back(p);
    CK(cudaMemsetAsync(p, 0, sizeof(T) * std::max<size_t>(count, 1), stream));
    return static_cast<T*>(p);
  }
  // drop the captured tick: its kernel arguments name buffers and shard bounds
  void invalidate_graph() {
    if (tick_exec) cudaGraphExecDestroy(tick_exec);
    if (tick_graph) cudaGraphDestroy(tick_graph);
    tick_exec = nullptr;
    tick_graph = nullptr;
    graph_key = -1;
  }
  ~gpmppi_planner() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : allocs) cudaFree(p);
    for (void* p : sample_allocs) cudaFree(p);
    if (h_x0) cudaFreeHost(h_x0);  // h_task lives in the same pinned block
    if (h_out) cudaFreeHost(h_out);
    if (h_infeasible) cudaFreeHost(h_infeasible);
    if (h_done) cudaFreeHost(h_done);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (tick_exec) cudaGraphExecDestroy(tick_exec);
    if (tick_graph) cudaGraphDestroy(tick_graph);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
    if (comm && nccl_api().comm_destroy) nccl_api().comm_destroy(comm);
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
  }
  long long slots() const { return (long long)B * K_local; }
  int groups() const { return model ? model->dev.G : 0; }
  // (Re)allocate every buffer sized by the local sample count; the previous set (if any)
  // is freed and the captured tick graph dropped (set_shard changes the count).
  void alloc_sample_buffers() {
    CK(cudaStreamSynchronize(stream));
    invalidate_graph();
    for (void* q : sample_allocs) CK(cudaFree(q));
    sample_allocs.clear();
    d_eps = nullptr;
    d_noise = nullptr;
    injected_set = false;
    d_queries = nullptr;
    d_var = nullptr;
    std::vector<void*>* o = &sample_allocs;
    const long long S = slots();
    d_cost_mean = dalloc<double>(S, o);
    d_costs = dalloc<double>(S, o);
    d_e = dalloc<double>(S, o);
    d_viol = dalloc<uint32_t>((size_t)S * words, o);
    d_coll = dalloc<uint32_t>((size_t)S * words, o);
    d_term = dalloc<uint8_t>(S, o);
    d_alive = dalloc<uint8_t>(S, o);
    // Philox noise materialised by the rollout for the reduce (16 B per sample-step written +
    // read) up to kNoiseMatMax sample-steps, else regenerated from the counter in the reduce.
    // Measured (profiles/r02/config5_sweep.md): the FP64 Box-Muller regeneration costs more
    // than the HBM round trip at every K up to 4M (reduce 4.46 vs 2.13 ms at K = 4M), so the
    // bound is the 2^31 sample-step planner limit. GPMPPI_NOISE_MAT=0/1 forces either.
    static const int mat_env = getenv("GPMPPI_NOISE_MAT") ? atoi(getenv("GPMPPI_NOISE_MAT")) : -1;
    const bool mat = mat_env >= 0 ? mat_env != 0 : (long long)S * T <= kNoiseMatMax;
    d_noise = mat ? dalloc<double>((size_t)S * T * 2, o) : nullptr;
    if (model_kind == GPMPPI_MODEL_GP_ENSEMBLE) {
      // The co-resident variance (variance_coop_kernel, GPMPPI_COOP=1) needs one kernel group
      // with the 3xFP16 operand, a rollout block of <= 7 warps (registers) and room for both
      // blocks' shared memory on an SM. Off by default: measured slower than the sequential
      // rollout -> variance_f16_kernel sequence (profiles/r02/coop_variance.md).
      static const int coop_env = getenv("GPMPPI_COOP") ? atoi(getenv("GPMPPI_COOP")) : 0;
      const gpm::GroupDev& g0 = model->dev.g[0];
      const bool coop_possible =
          GPM_COOP && coop_env != 0 && groups() == 1 && g0.tc_h && g0.tc_hmeta && g0.tc_np <= 256;
      geom = gpm::rollout_geometry((int)K_local, B, T, model->n, groups(), num_sms, coop_possible ? 7 : 8);
      coop_ok = false;
      if (coop_possible) {
        gpm::RolloutArgs ra{};
        ra.model = model->dev;
        ra.model_kind = model_kind;
        ra.T = T;
        ra.n_obs_max = gpm::kMaxObstacles;  // the worst per-tick robot view
        ra.R = R;
        ra.geom = geom;
        for (int st = 3; st >= 2 && !coop_ok; --st) {
          ra.smem_budget = (int)(228 * 1024 - 2048 - gpm::coop_smem_bytes(g0, st));
          ra.smem_budget = std::min(ra.smem_budget, 227 * 1024);
          if (gpm::rollout_launch_smem(ra, nullptr) <= (size_t)ra.smem_budget) {
            coop_ok = true;
            coop_budget = ra.smem_budget;
          }
        }
      }
      q_slots = gpm::query_slots(geom, B, T);  // item-major, padded to whole items
      d_queries = dalloc<float4>((size_t)q_slots, o);
      d_var = dalloc<double>((size_t)groups() * q_slots, o);
      progress_words = (long long)B * geom.chunks * (geom.threads / geom.lps);
      d_progress = dalloc<unsigned long long>((size_t)progress_words, o);
      if (!d_scratch) d_scratch = dalloc<double>(gpm::rollout_scratch_doubles(T, num_sms));
    }
    reduce_blocks = gpm::reduce_blocks_for((int)K_local, B, num_sms, T);
    d_partials = dalloc<double>((size_t)B * reduce_blocks * gpm::tuple_doubles(T), o);
  }
};

namespace {

// Host -> device update of planner state on the planner's own (non-blocking) stream, so it
// is ordered after every kernel already enqueued there; returns once the copy has landed
// (the source may be pageable and is reused by the caller).
void h2d_sync(gpmppi_planner* p, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, p->stream));
  CK(cudaStreamSynchronize(p->stream));
}

double normal_quantile(double p) {  // uncertainty.cpp:19-60 (Acklam + one Newton step)
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01,  -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  const double plow = 0.02425;
  double x;
  if (p < plow) {
    const double q = std::sqrt(-2.0 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p > 1.0 - plow) {
    const double q = std::sqrt(-2.0 * std::log(1.0 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  }
  const double pdf = std::exp(-0.5 * x * x) / std::sqrt(2.0 * gpm::kPi);
  if (pdf > 1e-300) x -= (0.5 * std::erfc(-x * 0.70710678118654752440) - p) / pdf;
  return x;
}

bool on_simplex(const double* w, int R, double tol) {  // core.hpp:107-111
  if (R <= 0) return false;
  double s = 0.0;
  for (int i = 0; i < R; ++i) s += w[i];
  if (std::fabs(s - 1.0) > tol) return false;
  for (int i = 0; i < R; ++i)
    if (!(w[i] >= -tol) || !(w[i] <= 1.0 + tol)) return false;
  return true;
}

void validate_task(const gpmppi_task* t) {
  if (!t) invalid("plan_step: null task");
  if (t->kind < 0 || t->kind > 2) invalid("plan_step: unknown task kind");
  if (t->kind != GPMPPI_TASK_AVOIDANCE) {
    if (!t->track) invalid("plan_step: tracking task needs a track");
    const gpmppi_track& k = *t->track;  // costs.cpp:44-60
    if (!(k.half_width > 0.0)) invalid("Track: half_width must be positive");
    if (k.is_circle) {
      if (!(k.radius > 0.0)) invalid("Track: circle radius must be positive");
    } else {
      if (k.n_waypoints < 2) invalid("Track: polyline needs at least 2 waypoints");
      if (k.n_waypoints > GPMPPI_MAX_WAYPOINTS) invalid("Track: too many waypoints for the device task");
      for (int i = 1; i < k.n_waypoints; ++i) {
        const double dx = k.waypoints[2 * i] - k.waypoints[2 * i - 2];
        const double dy = k.waypoints[2 * i + 1] - k.waypoints[2 * i - 1];
        if (std::sqrt(dx * dx + dy * dy) < 1e-12) invalid("Track: consecutive waypoints must be distinct");
      }
    }
  }
  if (t->kind != GPMPPI_TASK_TRACKING) {
    if (t->n_obstacles < 0) invalid("plan_step: avoidance task needs an obstacle list");
    if (t->n_obstacles > 0 && !t->obstacles) invalid("plan_step: avoidance task needs an obstacle list");
    if (t->n_obstacles > GPMPPI_MAX_OBSTACLES) invalid("plan_step: too many obstacles for the device task");
  }
  if (t->kind == GPMPPI_TASK_AVOIDANCE && !(t->high_cost > 0.0))
    invalid("terminal_cost: high_cost must be positive");
}

void fill_task(gpm::TaskDev& d, const gpmppi_task* t) {
  std::memset(&d, 0, sizeof d);
  d.kind = t->kind;
  if (t->kind != GPMPPI_TASK_AVOIDANCE) {
    const gpmppi_track& k = *t->track;
    d.is_circle = k.is_circle;
    d.cx = k.cx;
    d.cy = k.cy;
    d.radius = k.radius;
    d.half_width = k.half_width;
    d.closed = k.closed;
    d.n_wp = k.is_circle ? 0 : k.n_waypoints;
    for (int i = 0; i < d.n_wp; ++i) {
      d.wp[i][0] = k.waypoints[2 * i];
      d.wp[i][1] = k.waypoints[2 * i + 1];
    }
  }
  d.v_desired = t->v_desired;
  d.tw[0] = t->tracking.variance;
  d.tw[1] = t->tracking.deviation;
  d.tw[2] = t->tracking.slip;
  d.tw[3] = t->tracking.safety;
  d.tw[4] = t->tracking.speed;
  d.aw[0] = t->avoidance.variance;
  d.aw[1] = t->avoidance.obstacle;
  d.aw[2] = t->avoidance.stage;
  d.aw[3] = t->avoidance.terminal;
  d.goal[0] = t->goal[0];
  d.goal[1] = t->goal[1];
  d.goal[2] = t->goal[2];
  d.high_cost = t->high_cost;
  d.n_obs = t->kind == GPMPPI_TASK_TRACKING ? 0 : t->n_obstacles;
  for (int i = 0; i < d.n_obs; ++i)
    for (int c = 0; c < 3; ++c) d.obs[i][c] = t->obstacles[3 * i + c];
}

void check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw CudaError{e, where};
  static const int dbg_sync = getenv("GPMPPI_DEBUG_SYNC") ? atoi(getenv("GPMPPI_DEBUG_SYNC")) : 0;  // diagnostics
  if (dbg_sync) {
    const cudaError_t se = cudaDeviceSynchronize();
    if (se != cudaSuccess) throw CudaError{se, where};
  }
}

double task_var_weight(const gpmppi_task* t) {
  return t->kind == GPMPPI_TASK_AVOIDANCE ? t->avoidance.variance : t->tracking.variance;
}

void finish_pending(gpmppi_planner* p, gpmppi_diag* diag);

// mppi.cpp:235-248 ensure_thresholds + the per-tick staging of every robot's state,
// task, variance weight and Philox key into pinned memory (enqueue_h2d copies them).
void stage_tick(gpmppi_planner* p, const double* x0, const gpmppi_task* tasks) {
  NvtxRange nv("gpmppi:stage tick");
  if (!x0 || !tasks) invalid("plan_step: null state or task");
  const int T = p->T;
  for (int b = 0; b < p->B; ++b) {
    for (int i = 0; i < 5; ++i)
      if (!std::isfinite(x0[5 * b + i])) invalid("plan_step: non-finite state estimate");
    validate_task(&tasks[b]);
  }
  int omax = 0;
  bool synced = false;
  for (int b = 0; b < p->B; ++b) {
    const gpmppi_task* task = &tasks[b];
    if (task->kind != GPMPPI_TASK_AVOIDANCE && !p->rbar_init[b]) {
      if (!synced) {  // the pinned staging buffers may still feed the previous tick's copies
        CK(cudaStreamSynchronize(p->stream));
        synced = true;
      }
      std::vector<double> r(T, task->track->half_width);
      h2d_sync(p, p->d_rbar + (size_t)b * gpm::BatchStrides::rbar(T), r.data(), sizeof(double) * T);
      p->rbar_init[b] = 1;
    }
    const int O = task->kind == GPMPPI_TASK_TRACKING ? 0 : task->n_obstacles;
    if (task->kind != GPMPPI_TASK_TRACKING && p->margins_O[b] != O) {
      CK(cudaMemsetAsync(p->d_margins + (size_t)b * gpm::BatchStrides::marg(T), 0,
                         sizeof(double) * gpm::BatchStrides::marg(T), p->stream));
      p->margins_O[b] = O;
    }
    omax = std::max(omax, O);
  }
  finish_pending(p, nullptr);  // previous tick's staging copies (and tightening) are done
  for (int b = 0; b < p->B; ++b) {
    fill_task(p->h_task[b], &tasks[b]);
    double* blk = p->h_x0 + (size_t)b * gpm::BatchStrides::X0;
    for (int i = 0; i < 5; ++i) blk[i] = x0[5 * b + i];
    blk[5] = task_var_weight(&tasks[b]);
    const uint64_t key = gpm::philox_key(p->seeds[b], p->tick);
    std::memcpy(&blk[6], &key, sizeof key);
    blk[7] = p->seq + 1.0;  // this tick's sequence number (zero-copy completion words)
  }
  p->seq += 1.0;
  p->n_obs_max = omax;
}

// the tick's two H2D copies from the pinned staging buffers (captured in the tick graph)
void enqueue_h2d(gpmppi_planner* p) {  // tick blocks + tasks: one copy (contiguous on both sides)
  if (p->dh_x0)  // a staging kernel reads the mapped block (GPMPPI_H2D_COPY=1: a copy node)
    check(gpm::launch_stage_tick(p->dh_x0, p->d_x0, p->tick_bytes, p->stream), "stage tick");
  else
    CK(cudaMemcpyAsync(p->d_x0, p->h_x0, p->tick_bytes, cudaMemcpyHostToDevice, p->stream));
}

bool command_in_tightening(const gpmppi_planner* p);

// Rollout + variance + reduce for every robot's sample range. finish=1 also
// applies the update (single-rank solve).
void enqueue_samples(gpmppi_planner* p, int finish, cudaEvent_t* evs) {
  NvtxRange nv("gpmppi:enqueue rollout+variance+reduce");
  const int T = p->T;
  gpm::RolloutArgs a{};
  if (p->model) a.model = p->model->dev;
  a.model_kind = p->model_kind;
  a.nom = p->nom;
  a.edd5 = p->edd5;
  a.B = p->B;
  a.K_local = (int)p->K_local;
  a.K_total = p->K_total;
  a.s_begin = p->s_begin;
  a.T = T;
  a.n_obs_max = p->n_obs_max;
  a.lo[0] = p->cfg.lo[0];
  a.lo[1] = p->cfg.lo[1];
  a.hi[0] = p->cfg.hi[0];
  a.hi[1] = p->cfg.hi[1];
  a.sv = std::sqrt(p->cfg.sigma_v2);
  a.sw = std::sqrt(p->cfg.sigma_w2);
  a.noise_mode = p->noise_mode;
  a.eps = p->d_eps;
  a.noise_out = p->noise_mode == gpm::NOISE_PHILOX ? p->d_noise : nullptr;
  a.nominal_seq = p->d_nom;
  a.tw = p->d_tw;
  a.R = p->R;
  a.task = p->d_task;
  a.r_bar = p->d_rbar;
  a.margins = p->d_margins;
  a.x0 = p->d_x0;
  a.cost_mean = p->d_cost_mean;
  a.queries = p->d_queries;
  a.viol_bits = p->d_viol;
  a.coll_bits = p->d_coll;
  a.term = p->d_term;
  a.alive = p->d_alive;
  a.words = p->words;
  a.scratch = p->d_scratch;
  a.geom = p->geom;
  const bool gp = p->model_kind == GPMPPI_MODEL_GP_ENSEMBLE;
  // concurrent variance: the rollout publishes its query progress, the variance kernel
  // launches as its programmatic dependent and shares the SMs (phase events would split
  // them, so the per-phase timing pass keeps the sequential path)
  const bool coop = gp && p->coop_ok && p->var_path == GPMPPI_VAR_TC_3XF16 && !evs;
  a.progress = coop ? p->d_progress : nullptr;
  a.smem_budget = coop ? p->coop_budget : 0;
  if (evs) CK(cudaEventRecord(evs[0], p->stream));
  check(gpm::launch_rollout(a, p->num_sms, p->stream), "rollout kernel");
  if (evs) CK(cudaEventRecord(evs[1], p->stream));
  const long long KT = p->q_slots;  // item-major query / trace slots
  if (coop) {
    gpm::VarianceArgs v{};
    v.queries = p->d_queries;
    v.KT = KT;
    v.n = p->model->n;
    v.g = p->model->dev.g[0];
    v.coef = 1.0;
    v.accumulate = 0;
    v.trace = p->d_var;
    check(gpm::launch_variance_coop(v, p->d_progress, p->progress_words, T, p->geom,
                                    gpm::rollout_launch_smem(a, nullptr), p->num_sms, p->stream),
          "co-resident variance kernel");
  } else if (gp) {
    for (int g = 0; g < p->groups(); ++g) {  // raw variances; the reduce applies Σ w² per robot
      gpm::VarianceArgs v{};
      v.queries = p->d_queries;
      v.KT = KT;
      v.n = p->model->n;
      v.g = p->model->dev.g[g];
      v.coef = 1.0;
      v.accumulate = 0;
      v.trace = p->d_var + (size_t)g * KT;
      check(gpm::launch_variance(v, p->var_path, p->stream), "variance kernel");
    }
  }
  if (evs) CK(cudaEventRecord(evs[2], p->stream));
  gpm::ReduceArgs r{};
  r.geom = p->geom;
  r.progress = coop ? p->d_progress : nullptr;
  r.progress_words = p->progress_words;
  r.B = p->B;
  r.K_local = (int)p->K_local;
  r.K_total = p->K_total;
  r.s_begin = p->s_begin;
  r.T = T;
  r.bpr = p->reduce_blocks;
  r.lambda = p->cfg.lambda;
  r.cost_mean = p->d_cost_mean;
  r.var = gp ? p->d_var : nullptr;
  r.G = gp ? p->groups() : 0;
  r.tw = p->d_tw;
  r.x0 = p->d_x0;
  // Philox mode: the rollout materialised the noise, so the reduce reads it like injected noise
  r.noise_mode = p->d_noise && p->noise_mode == gpm::NOISE_PHILOX ? gpm::NOISE_INJECTED : p->noise_mode;
  r.eps = p->noise_mode == gpm::NOISE_PHILOX ? p->d_noise : p->d_eps;  // null: regenerated from the counter
  r.sv = a.sv;
  r.sw = a.sw;
  r.costs_out = p->d_costs;
  r.e_out = p->d_e;
  r.partials = p->d_partials;
  r.ticket = p->d_ticket;
  r.rank_tuple = p->d_rank_tuple;
  r.finish = finish;
  r.nominal_seq = p->d_nom;
  r.lo[0] = p->cfg.lo[0];
  r.lo[1] = p->cfg.lo[1];
  r.hi[0] = p->cfg.hi[0];
  r.hi[1] = p->cfg.hi[1];
  r.out = p->d_out;
  r.out_host = p->zc_tick && !command_in_tightening(p) ? p->d_out_host : nullptr;
  check(gpm::launch_reduce(r, p->B * p->reduce_blocks, p->stream), "reduce kernel");
  if (evs) CK(cudaEventRecord(evs[3], p->stream));
}

// Samples + update of one tick. Single rank: the reduce's last CTA applies the update.
// Sharded (NCCL attached): the reduce leaves this rank's tuple, one ncclAllGather on the
// planner stream exchanges the (2T+6)-double tuples, and finish_kernel
// combines them in rank order and applies update / clamp / shift identically on every
// rank -- no host synchronisation between the rollout and the command.
void enqueue_update(gpmppi_planner* p, cudaEvent_t* evs) {
  if (!p->comm) {
    enqueue_samples(p, 1, evs);
    return;
  }
  enqueue_samples(p, 0, evs);
  const int W = gpm::tuple_doubles(p->T);
  nccl_check(nccl_api().all_gather(p->d_rank_tuple, p->d_gathered, (size_t)W, ncclDouble, p->comm, p->stream),
             "ncclAllGather");
  check(gpm::launch_finish(p->d_gathered, p->n_ranks, p->T, p->cfg.lambda, p->d_nom, p->cfg.lo, p->cfg.hi,
                           p->d_out, p->K_total, p->d_combined, p->stream, p->zc_tick ? p->d_out_host : nullptr,
                           p->d_x0),
        "finish kernel");
  if (evs) CK(cudaEventRecord(evs[3], p->stream));  // the exchange counts to the reduce phase
}

// single-robot GP planners run the pipelined tightening pass (TightenArgs::tflags)
bool pipelined_tightening(const gpmppi_planner* p) {
  static const int seq_env = getenv("GPMPPI_TIGHTEN_SEQUENTIAL") ? atoi(getenv("GPMPPI_TIGHTEN_SEQUENTIAL")) : 0;
  return p->B == 1 && p->model_kind == GPMPPI_MODEL_GP_ENSEMBLE && !seq_env;
}
// ... and then the mean kernel's publisher warp, not the reduce's last block, writes the
// command into the mapped words: the system-scope fence leaves the tick's critical path
// (only when plan_step waits for the whole tick: in command-first mode the reduce publishes,
// ~2 us sooner to the command; measured 0.3707 vs 0.3722 ms full plan_step, 0.3362 vs 0.3338
// command-first at config 2)
bool command_in_tightening(const gpmppi_planner* p) {
  static const int env = getenv("GPMPPI_CMD_IN_TIGHTEN") ? atoi(getenv("GPMPPI_CMD_IN_TIGHTEN")) : 1;
  return env && p->zc_tick && !p->comm && !p->command_first && pipelined_tightening(p);
}

void enqueue_tighten(gpmppi_planner* p) {
  NvtxRange nv("gpmppi:enqueue tightening");
  gpm::TightenArgs t{};
  if (p->model) t.model = p->model->dev;
  t.model_kind = p->model_kind;
  t.nom = p->nom;
  t.B = p->B;
  t.T = p->T;
  t.tw = p->d_tw;
  t.R = p->R;
  t.x0 = p->d_x0;
  t.nominal_seq = p->d_nom;
  t.task = p->d_task;
  t.chi2 = p->chi2;
  t.z = p->z;
  t.horizon_cov = p->d_hcov;
  t.r_bar = p->d_rbar;
  t.margins = p->d_margins;
  t.infeasible = p->d_infeasible;
  t.tq = p->d_tq;
  t.tmu = p->d_tmu;
  t.tJ = p->d_tJ;
  t.tvar_part = p->d_tvar;
  t.done_host = p->zc_tick ? p->d_done_host : nullptr;
  t.tflags = pipelined_tightening(p) ? p->d_tflags : nullptr;
  t.tcv = p->d_tcv;
  t.cmd_host = command_in_tightening(p) ? p->d_out_host : nullptr;
  t.cmd_dev = p->d_out;
  check(gpm::launch_tighten(t, p->stream), "tighten kernel");
}

void copy_out_async(gpmppi_planner* p) {  // command + diagnostics of every robot
  CK(cudaMemcpyAsync(p->h_out, p->d_out, sizeof(double) * gpm::BatchStrides::OUT * p->B,
                     cudaMemcpyDeviceToHost, p->stream));
}

void fill_diag(gpmppi_planner* p, double* command, gpmppi_diag* diag, double t_cmd, double t_all) {
  for (int b = 0; b < p->B; ++b) {
    const double* o = p->h_out + (size_t)b * gpm::BatchStrides::OUT;
    command[2 * b] = o[0];
    command[2 * b + 1] = o[1];
    if (diag) {
      gpmppi_diag& d = diag[b];
      d.best_cost = o[2];
      d.mean_cost = o[3];
      d.ess = o[4];
      d.weight_entropy = o[5];
      d.nonfinite_samples = (int)o[6];
      d.tightening_infeasible = p->zero_copy ? (int)p->h_done[2 * b] : p->h_infeasible[b];
      d.plan_ms = t_all;
      d.command_ms = t_cmd;
    }
  }
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

void upload_terrain_weights(gpmppi_planner* p) {
  std::vector<double> w((size_t)p->B * gpm::BatchStrides::TW, 0.0);
  for (int b = 0; b < p->B; ++b) {
    double* row = &w[(size_t)b * gpm::BatchStrides::TW];
    for (int i = 0; i < p->R; ++i) row[i] = p->tw[(size_t)b * p->R + i];
    // variance trace coefficient of each kernel group: Σ over the group's outputs (ascending)
    // of w(terrain of the output)² -- ensemble_combine's Σ w_i² var (gp.cpp:380-386)
    for (int g = 0; g < p->groups(); ++g) {
      const gpm::GroupDev& G = p->model->dev.g[g];
      double c = 0.0;
      for (int o = 0; o < G.n_out; ++o) {
        const double wi = row[G.out_idx[o] >> 1];
        c = std::fma(wi, wi, c);
      }
      row[gpm::BatchStrides::TW_COEF + g] = c;
    }
  }
  h2d_sync(p, p->d_tw, w.data(), sizeof(double) * w.size());
}

gpmppi_planner* create_planner(const gpmppi_mppi_config* cfg, const gpmppi_prediction_model* pm,
                               const gpmppi_nominal* nominal, double p_x, int n_robots,
                               const uint64_t* seeds, int device) {
  if (!cfg || !pm || !nominal) invalid("Planner: null argument");
  if (!(p_x > 0.5) || !(p_x < 1.0)) invalid("QuantileTables: p_x must lie in (0.5, 1)");
  if (cfg->samples < 1 || cfg->horizon < 1) invalid("MppiConfig: samples and horizon must be >= 1");
  if (!(cfg->lambda > 0.0)) invalid("MppiConfig: lambda must be positive");
  if (!(cfg->sigma_v2 > 0.0) || !(cfg->sigma_w2 > 0.0))
    invalid("MppiConfig: sampling variances must be positive");
  if (cfg->lo[0] >= cfg->hi[0] || cfg->lo[1] >= cfg->hi[1])
    invalid("MppiConfig: control bounds must be a nonempty box");
  if (!(nominal->tau_v > 0.0) || !(nominal->tau_omega > 0.0))
    invalid("NominalParams: time constants must be positive");
  if (!(nominal->dt > 0.0) || nominal->dt >= std::min(nominal->tau_v, nominal->tau_omega))
    invalid("NominalParams: require 0 < dt < min(tau_v, tau_omega)");
  if (pm->kind < 0 || pm->kind > 3) invalid("Planner: unknown prediction model");
  if (pm->kind == GPMPPI_MODEL_GP_ENSEMBLE &&
      (pm->gp == nullptr || pm->n_terrains < 1 || pm->gp->m != 2 * pm->n_terrains))
    invalid("Planner: GP ensemble needs a model with 2M outputs");
  if (pm->kind == GPMPPI_MODEL_GP_ENSEMBLE && pm->n_terrains > gpm::kMaxTerrains)
    invalid("Planner: too many terrains for the device planner");
  if (pm->kind == GPMPPI_MODEL_EDD5) {
    if (!(pm->track_width > 0.0)) invalid("step_edd5: track_width must be positive");
    if (pm->edd5.y_icr_r - pm->edd5.y_icr_l <= 1e-6)
      invalid("step_edd5: degenerate ICR span (y_icr_r - y_icr_l <= 1e-6)");
  }
  if (n_robots < 1) invalid("Planner: robot count must be >= 1");
  if ((long long)n_robots * cfg->samples * cfg->horizon > (1LL << 31) - 1)
    invalid("Planner: robots x samples x horizon exceeds 2^31 sample-steps");
  require_device(device);
  auto* p = new gpmppi_planner();
  try {
    p->device = device;
    CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&p->fork_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->join_ev, cudaEventDisableTiming));
    CK(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device));
    p->cfg = *cfg;
    p->B = n_robots;
    p->seeds.resize(n_robots);
    for (int b = 0; b < n_robots; ++b) p->seeds[b] = seeds ? seeds[b] : cfg->seed + (uint64_t)b;
    p->model_kind = pm->kind;
    p->model = pm->kind == GPMPPI_MODEL_GP_ENSEMBLE ? pm->gp : nullptr;
    if (p->model && p->model->device != device) invalid("Planner: GP model lives on another device");
    p->R = pm->kind == GPMPPI_MODEL_GP_ENSEMBLE ? pm->n_terrains : 1;
    p->edd5 = {pm->edd5.alpha_l, pm->edd5.alpha_r, pm->edd5.x_icr, pm->edd5.y_icr_l,
               pm->edd5.y_icr_r, pm->track_width};
    p->nom = {nominal->tau_v, nominal->tau_omega, nominal->dt};
    p->p_x = p_x;
    p->chi2 = -2.0 * std::log1p(-p_x);  // uncertainty.cpp:8-13
    p->z = normal_quantile(p_x);
    p->tw.assign((size_t)n_robots * p->R, 1.0 / p->R);
    p->T = cfg->horizon;
    p->words = (p->T + 31) / 32;
    p->K_total = cfg->samples;
    p->K_local = cfg->samples;
    p->s_begin = 0;
    p->rbar_init.assign(n_robots, 0);
    p->margins_O.assign(n_robots, -1);
    const int T = p->T, B = n_robots;
    p->d_nom = p->dalloc<double>((size_t)B * 2 * T);
    std::vector<double> nom0((size_t)B * 2 * T);  // bounds.clamp(Control{}) (mppi.cpp:200)
    for (size_t k = 0; k < (size_t)B * T; ++k) {
      nom0[2 * k] = gpm::clampd(0.0, cfg->lo[0], cfg->hi[0]);
      nom0[2 * k + 1] = gpm::clampd(0.0, cfg->lo[1], cfg->hi[1]);
    }
    CK(cudaMemcpyAsync(p->d_nom, nom0.data(), sizeof(double) * nom0.size(), cudaMemcpyHostToDevice, p->stream));
    p->d_tw = p->dalloc<double>((size_t)B * gpm::BatchStrides::TW);
    upload_terrain_weights(p);
    // tick blocks [B][8] and tasks [B] in one device block (and one pinned block): the tick's
    // inputs move in a single H2D copy
    const size_t x0_bytes = sizeof(double) * gpm::BatchStrides::X0 * B;
    p->tick_bytes = x0_bytes + sizeof(gpm::TaskDev) * B;
    unsigned char* dblk = p->dalloc<unsigned char>(p->tick_bytes);
    p->d_x0 = reinterpret_cast<double*>(dblk);
    p->d_rbar = p->dalloc<double>((size_t)B * gpm::BatchStrides::rbar(T));
    p->d_margins = p->dalloc<double>((size_t)B * gpm::BatchStrides::marg(T));
    p->d_task = reinterpret_cast<gpm::TaskDev*>(dblk + x0_bytes);
    p->d_rank_tuple = p->dalloc<double>((size_t)B * gpm::tuple_doubles(T));
    p->d_combined = p->dalloc<double>(gpm::tuple_doubles(T));
    p->d_out = p->dalloc<double>((size_t)B * gpm::BatchStrides::OUT);
    p->d_hcov = p->dalloc<double>((size_t)B * T * 25);
    p->d_ticket = p->dalloc<unsigned int>(B);
    p->d_infeasible = p->dalloc<int>(B);
    p->d_tq = p->dalloc<double>((size_t)B * T * 4);
    p->d_tflags = p->dalloc<unsigned int>((size_t)T + 2);  // query count, J count, per-step variance counts
    CK(cudaMemsetAsync(p->d_tflags, 0, sizeof(unsigned int) * ((size_t)T + 2), p->stream));
    p->d_tcv = p->dalloc<double>((size_t)2 * T);
    p->d_tmu = p->dalloc<double>((size_t)B * (T + 1) * 5);
    p->d_tJ = p->dalloc<double>((size_t)B * T * 25);
    {
      const int G = p->model ? p->groups() : 1;
      const int ns = p->model ? gpm::tighten_splits(p->model->n, B) : 1;
      p->d_tvar = p->dalloc<double>((size_t)B * T * G * ns);
    }
    p->alloc_sample_buffers();
    CK(cudaHostAlloc(&p->h_x0, p->tick_bytes, cudaHostAllocMapped));
    {
      static const int copy_env = getenv("GPMPPI_H2D_COPY") ? atoi(getenv("GPMPPI_H2D_COPY")) : 0;
      double* dp = nullptr;
      if (!copy_env && cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), p->h_x0, 0) == cudaSuccess)
        p->dh_x0 = dp;
      cudaGetLastError();
    }
    p->h_task = reinterpret_cast<gpm::TaskDev*>(reinterpret_cast<unsigned char*>(p->h_x0) + x0_bytes);
    CK(cudaHostAlloc(&p->h_out, sizeof(double) * gpm::BatchStrides::OUT * B, cudaHostAllocMapped));
    CK(cudaHostAlloc(&p->h_done, sizeof(double) * 2 * B, cudaHostAllocMapped));
    std::memset(p->h_out, 0, sizeof(double) * gpm::BatchStrides::OUT * B);
    std::memset(p->h_done, 0, sizeof(double) * 2 * B);
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->d_out_host), p->h_out, 0));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->d_done_host), p->h_done, 0));
    CK(cudaMallocHost(&p->h_infeasible, sizeof(int) * B));
    for (auto& e : p->ev) CK(cudaEventCreate(&e));
    CK(cudaStreamSynchronize(p->stream));
  } catch (...) {
    delete p;
    throw;
  }
  return p;
}

// The device work of one tick after staging: H2D, samples + update, command D2H (event
// ev[0] marks the command), tightening (mppi.cpp:433), infeasibility D2H.
void enqueue_tick(gpmppi_planner* p, bool capturing) {
  auto rec = [&](cudaEvent_t e, cudaStream_t st) {
    if (capturing)
      CK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else
      CK(cudaEventRecord(e, st));
  };
  rec(p->ev[1], p->stream);  // device start of the tick (plan_ms in command-first mode)
  enqueue_h2d(p);
  if (p->zero_copy) {
    // the reduce (or finish) kernel and the covariance kernel publish into mapped pinned
    // memory; no copies or events sit between the tick's kernels and the host
    p->zc_tick = true;
    try {
      enqueue_update(p, nullptr);
      enqueue_tighten(p);
    } catch (...) {
      p->zc_tick = false;
      throw;
    }
    p->zc_tick = false;
    rec(p->ev[2], p->stream);
    return;
  }
  enqueue_update(p, nullptr);
  // the command / diagnostics readback forks off onto the side stream, so the tightening
  // follows the reduction directly on the main stream (no copy on its critical path)
  CK(cudaEventRecord(p->fork_ev, p->stream));
  CK(cudaStreamWaitEvent(p->side, p->fork_ev, 0));
  CK(cudaMemcpyAsync(p->h_out, p->d_out, sizeof(double) * gpm::BatchStrides::OUT * p->B, cudaMemcpyDeviceToHost,
                     p->side));
  rec(p->ev[0], p->side);
  CK(cudaEventRecord(p->join_ev, p->side));
  enqueue_tighten(p);
  CK(cudaStreamWaitEvent(p->stream, p->join_ev, 0));
  CK(cudaMemcpyAsync(p->h_infeasible, p->d_infeasible, sizeof(int) * p->B, cudaMemcpyDeviceToHost, p->stream));
  rec(p->ev[2], p->stream);  // tightening and its readback done
}

// Spin until every robot's completion word (stride doubles apart, at `slot`) carries this
// tick's sequence number. The stream is queried every few thousand spins so a failed
// kernel surfaces as its CUDA error instead of a hang.
void wait_host_words(gpmppi_planner* p, const double* words, int stride, int slot, const char* what) {
  const volatile double* w = words;
  for (unsigned it = 1;; ++it) {
    bool all = true;
    for (int b = 0; b < p->B && all; ++b) all = w[(size_t)b * stride + slot] == p->seq;
    if (all) return;
    if ((it & 4095u) == 0) {
      const cudaError_t e = cudaStreamQuery(p->stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) throw CudaError{e, what};
      if (e == cudaSuccess) {  // stream drained: the words must be there now
        for (int b = 0; b < p->B; ++b)
          if (w[(size_t)b * stride + slot] != p->seq) runtime(std::string(what) + ": completion word missing");
        return;
      }
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
}

// Capture the tick into a graph (one launch instead of eight stream operations). Any
// capture failure leaves the planner on the per-operation path.
void capture_tick(gpmppi_planner* p, long long key) {
  if (p->tick_exec) cudaGraphExecDestroy(p->tick_exec);
  if (p->tick_graph) cudaGraphDestroy(p->tick_graph);
  p->tick_exec = nullptr;
  p->tick_graph = nullptr;
  const unsigned long long l0 = gpm::launches_total();
  bool ok = cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    try {
      enqueue_tick(p, true);
    } catch (...) {
      ok = false;
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(p->stream, &g);
    ok = ok && e == cudaSuccess && g != nullptr;
    if (ok) {
      p->tick_graph = g;
      ok = cudaGraphInstantiate(&p->tick_exec, g, 0) == cudaSuccess;
    } else if (g) {
      cudaGraphDestroy(g);
    }
  }
  const int n = (int)(gpm::launches_total() - l0);  // counted while capturing, launched on replay
  gpm::count_launch(-n);
  cudaGetLastError();  // clear a failed capture's error state
  if (!ok) {
    if (p->tick_exec) cudaGraphExecDestroy(p->tick_exec);
    p->tick_exec = nullptr;
    p->use_graph = false;
    return;
  }
  p->graph_launches = n;
  p->graph_key = key;
}

// One tick of every robot: mppi.cpp:389-462 (plan_step_impl) for B planners at once.
void plan_tick(gpmppi_planner* p, const double* x0, const gpmppi_task* tasks, double* command,
               gpmppi_diag* diag) {
  const auto t0 = Clock::now();  // mppi.cpp:391
  NvtxRange nv("gpmppi:plan_step");
  CK(cudaSetDevice(p->device));
  if (!command) invalid("plan_step: null command output");
  if (p->K_local != p->K_total && !p->comm)
    invalid("plan_step: sharded planner without a communicator; attach one or use plan_partial/plan_finish");
  if (p->noise_mode == gpm::NOISE_INJECTED && !p->injected_set) invalid("plan_step: injected noise mode without noise");
  stage_tick(p, x0, tasks);
  // everything a captured kernel argument depends on (device buffers are fixed per planner)
  const long long key = (long long)p->n_obs_max | ((long long)p->noise_mode << 8) | ((long long)p->var_path << 10) |
                        ((long long)p->R << 16) | ((long long)(p->comm != nullptr) << 24) |
                        ((long long)p->command_first << 25);  // who publishes the command (command_in_tightening)
  if (p->use_graph && (!p->tick_exec || p->graph_key != key)) capture_tick(p, key);
  if (p->use_graph && p->tick_exec) {
    CK(cudaGraphLaunch(p->tick_exec, p->stream));
    gpm::count_launch(p->graph_launches);
  } else {
    enqueue_tick(p, false);
  }
  const double t_launch = ms_since(t0);
  {
    NvtxRange wait("gpmppi:wait command");
    if (p->zero_copy)
      wait_host_words(p, p->h_out, gpm::BatchStrides::OUT, gpm::BatchStrides::OUT - 1, "plan_step (command)");
    else
      CK(cudaEventSynchronize(p->ev[0]));
  }
  const double t_cmd = ms_since(t0);
  if (p->command_first) {
    // command and diagnostics are on the host; the tightening (next tick's thresholds)
    // finishes behind the return. stage_tick / accessors / wait_tightening wait for it.
    p->pending_diag.assign(p->B, gpmppi_diag{});
    fill_diag(p, command, p->pending_diag.data(), t_cmd, t_cmd);  // h_infeasible is still in flight
    for (int b = 0; b < p->B; ++b) {
      p->pending_diag[b].tightening_infeasible = 0;  // known at completion
      p->pending_diag[b].plan_ms = t_launch;         // + device span at completion
    }
    if (diag)
      for (int b = 0; b < p->B; ++b) diag[b] = p->pending_diag[b];
    p->tightening_pending = true;
  } else {
    {
      NvtxRange wait("gpmppi:wait tightening");
      if (p->zero_copy)
        wait_host_words(p, p->h_done, 2, 1, "plan_step (tightening)");
      else
        CK(cudaStreamSynchronize(p->stream));
    }
    fill_diag(p, command, diag, t_cmd, ms_since(t0));
  }
  ++p->tick;  // mppi.cpp:460
}

// command-first mode: wait for the last tick's tightening and complete its diagnostics
// (tightening_infeasible, plan_ms = host launch latency + device span of the whole tick)
void finish_pending(gpmppi_planner* p, gpmppi_diag* diag) {
  CK(cudaStreamSynchronize(p->stream));
  if (!p->tightening_pending) return;
  p->tightening_pending = false;
  float dev_ms = 0.f;
  if (cudaEventElapsedTime(&dev_ms, p->ev[1], p->ev[2]) != cudaSuccess) dev_ms = 0.f;
  for (int b = 0; b < p->B; ++b) {
    gpmppi_diag& d = p->pending_diag[b];
    d.tightening_infeasible = p->zero_copy ? (int)p->h_done[2 * b] : p->h_infeasible[b];
    d.plan_ms = std::max(d.plan_ms + (double)dev_ms, d.command_ms);
    if (diag) diag[b] = d;
  }
}

void set_weights(gpmppi_planner* p, int robot, const double* w, int R) {  // mppi.cpp:208-218
  if (!w) invalid("set_terrain_weights: null weights");
  if (p->model_kind == GPMPPI_MODEL_GP_ENSEMBLE && R != p->R)
    invalid("set_terrain_weights: size mismatch with terrain count");
  if (!on_simplex(w, R, 1e-6)) invalid("set_terrain_weights: weights must lie on the simplex");
  if (R > gpm::kMaxTerrains) invalid("set_terrain_weights: too many terrains");
  if (R != p->R) {  // GP-free models carry weights they never use; keep every robot's row
    std::vector<double> nw((size_t)p->B * R, 1.0 / R);
    p->tw.swap(nw);
    p->R = R;
  }
  for (int b = 0; b < p->B; ++b)
    if (robot < 0 || robot == b) std::copy(w, w + R, p->tw.begin() + (size_t)b * R);
  upload_terrain_weights(p);
}

}  // namespace

extern "C" {

int gpmppi_planner_create(const gpmppi_mppi_config* cfg, const gpmppi_prediction_model* pm,
                          const gpmppi_nominal* nominal, double p_x, int device,
                          gpmppi_planner** out) {
  if (!out) return fail(GPMPPI_INVALID_ARGUMENT, "null output handle");
  *out = nullptr;
  return guarded([&] { *out = create_planner(cfg, pm, nominal, p_x, 1, nullptr, device); });
}

int gpmppi_planner_create_batch(const gpmppi_mppi_config* cfg, const gpmppi_prediction_model* pm,
                                const gpmppi_nominal* nominal, double p_x, int n_robots,
                                const uint64_t* seeds, int device, gpmppi_planner** out) {
  if (!out) return fail(GPMPPI_INVALID_ARGUMENT, "null output handle");
  *out = nullptr;
  return guarded([&] { *out = create_planner(cfg, pm, nominal, p_x, n_robots, seeds, device); });
}

void gpmppi_planner_free(gpmppi_planner* p) { delete p; }

int gpmppi_planner_robots(const gpmppi_planner* p) { return p ? p->B : 0; }

int gpmppi_planner_plan_step(gpmppi_planner* p, const double x0[5], const gpmppi_task* task,
                             double command[2], gpmppi_diag* diag) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    if (p->B != 1) invalid("plan_step: batched planner; use plan_step_batch");
    plan_tick(p, x0, task, command, diag);
  });
}

int gpmppi_planner_plan_step_batch(gpmppi_planner* p, const double* x0, const gpmppi_task* tasks,
                                   double* commands, gpmppi_diag* diags) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] { plan_tick(p, x0, tasks, commands, diags); });
}

int gpmppi_planner_set_terrain_weights(gpmppi_planner* p, const double* w, int R) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] { set_weights(p, -1, w, R); });
}

int gpmppi_planner_set_robot_terrain_weights(gpmppi_planner* p, int robot, const double* w, int R) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    if (robot < 0 || robot >= p->B) invalid("set_robot_terrain_weights: robot index out of range");
    set_weights(p, robot, w, R);
  });
}

int gpmppi_planner_terrain_weights(const gpmppi_planner* p, double* w) {
  if (!p) return 0;
  if (w) std::memcpy(w, p->tw.data(), sizeof(double) * p->tw.size());
  return p->R;
}

static int copy_back(const gpmppi_planner* p, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    CK(cudaSetDevice(p->device));
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, p->stream));  // after the tick's kernels
    CK(cudaStreamSynchronize(p->stream));
  });
}

int gpmppi_planner_nominal_sequence(const gpmppi_planner* p, double* seq) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return copy_back(p, seq, p->d_nom, sizeof(double) * 2 * p->T * p->B);
}
int gpmppi_planner_set_nominal_sequence(gpmppi_planner* p, const double* seq) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    h2d_sync(p, p->d_nom, seq, sizeof(double) * 2 * p->T * p->B);
  });
}
int gpmppi_planner_horizon_covariances(const gpmppi_planner* p, double* cov) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return copy_back(p, cov, p->d_hcov, sizeof(double) * 25 * p->T * p->B);
}
int gpmppi_planner_lane_radii(const gpmppi_planner* p, double* r) {
  if (!p) return 0;
  bool any = false;  // robots without a track keep zero rows
  for (int b = 0; b < p->B; ++b) any = any || p->rbar_init[b];
  if (!any) return 0;
  if (r && copy_back(p, r, p->d_rbar, sizeof(double) * p->T * p->B) != GPMPPI_OK) return -1;
  return p->T;
}
int gpmppi_planner_obstacle_margins(const gpmppi_planner* p, double* m) {
  if (!p) return 0;
  int O = 0;
  for (int b = 0; b < p->B; ++b) O = std::max(O, p->margins_O[b]);
  if (O <= 0) return 0;
  if (m) {
    const size_t stride = gpm::BatchStrides::marg(p->T);
    std::vector<double> tmp((size_t)p->B * stride);
    if (copy_back(p, tmp.data(), p->d_margins, sizeof(double) * tmp.size()) != GPMPPI_OK) return -1;
    for (int b = 0; b < p->B; ++b) {  // robot b's [T][O_b] block, zero-padded to O columns
      const int Ob = std::max(p->margins_O[b], 0);
      for (int k = 0; k < p->T; ++k)
        for (int o = 0; o < O; ++o)
          m[((size_t)b * p->T + k) * O + o] = o < Ob ? tmp[b * stride + (size_t)k * Ob + o] : 0.0;
    }
  }
  return O;
}
int gpmppi_planner_set_thresholds(gpmppi_planner* p, const double* r_bar, const double* margins,
                                  int n_obstacles) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    if (n_obstacles < 0 || n_obstacles > gpm::kMaxObstacles) invalid("set_thresholds: bad obstacle count");
    CK(cudaStreamSynchronize(p->stream));
    for (int b = 0; b < p->B; ++b) {
      if (r_bar) {
        h2d_sync(p, p->d_rbar + (size_t)b * gpm::BatchStrides::rbar(p->T), r_bar + (size_t)b * p->T,
                 sizeof(double) * p->T);
        p->rbar_init[b] = 1;
      }
      if (margins) {
        h2d_sync(p, p->d_margins + (size_t)b * gpm::BatchStrides::marg(p->T),
                 margins + (size_t)b * p->T * n_obstacles, sizeof(double) * p->T * n_obstacles);
        p->margins_O[b] = n_obstacles;
      }
    }
  });
}
uint64_t gpmppi_planner_tick(const gpmppi_planner* p) { return p ? p->tick : 0; }
int gpmppi_planner_horizon(const gpmppi_planner* p) { return p ? p->T : 0; }
int gpmppi_planner_samples(const gpmppi_planner* p) { return p ? (int)p->K_local : 0; }

int gpmppi_planner_set_noise_mode(gpmppi_planner* p, int mode) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  if (mode != GPMPPI_NOISE_PHILOX && mode != GPMPPI_NOISE_INJECTED) return fail(GPMPPI_INVALID_ARGUMENT, "unknown noise mode");
  p->noise_mode = mode;
  return GPMPPI_OK;
}
int gpmppi_planner_inject_noise(gpmppi_planner* p, const double* eps) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    const size_t cnt = (size_t)p->slots() * p->T * 2;
    if (!p->d_eps) {
      p->d_eps = p->dalloc<double>(cnt, &p->sample_allocs);
      p->invalidate_graph();  // the captured rollout / reduce name the injected buffer
    }
    h2d_sync(p, p->d_eps, eps, sizeof(double) * cnt);
    p->injected_set = true;
    p->noise_mode = gpm::NOISE_INJECTED;
  });
}
int gpmppi_planner_philox_noise(const gpmppi_planner* p, uint64_t tick, double* eps) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    CK(cudaSetDevice(p->device));
    double* d = nullptr;
    const size_t cnt = (size_t)p->K_local * p->T * 2;
    CK(cudaMalloc(&d, sizeof(double) * cnt));
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < p->B && e == cudaSuccess; ++b) {
      e = gpm::launch_philox_noise(gpm::philox_key(p->seeds[b], tick), p->s_begin, (int)p->K_local, p->T,
                                   std::sqrt(p->cfg.sigma_v2), std::sqrt(p->cfg.sigma_w2), d, p->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
      if (e == cudaSuccess) e = cudaMemcpy(eps + b * cnt, d, sizeof(double) * cnt, cudaMemcpyDeviceToHost);
    }
    cudaFree(d);
    if (e != cudaSuccess) throw CudaError{e, "philox_noise_kernel"};
  });
}

int gpmppi_planner_sample_costs(const gpmppi_planner* p, double* costs) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return copy_back(p, costs, p->d_costs, sizeof(double) * p->slots());
}
int gpmppi_planner_sample_weights(const gpmppi_planner* p, double* w) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    CK(cudaSetDevice(p->device));
    CK(cudaStreamSynchronize(p->stream));
    const int W = gpm::tuple_doubles(p->T);
    const int BP = p->reduce_blocks;
    std::vector<double> e(p->slots()), parts((size_t)p->B * BP * W), tup((size_t)p->B * W);
    CK(cudaMemcpy(e.data(), p->d_e, sizeof(double) * e.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(parts.data(), p->d_partials, sizeof(double) * parts.size(), cudaMemcpyDeviceToHost));
    if (p->K_local == p->K_total)
      CK(cudaMemcpy(tup.data(), p->d_rank_tuple, sizeof(double) * tup.size(), cudaMemcpyDeviceToHost));
    else
      CK(cudaMemcpy(tup.data(), p->d_combined, sizeof(double) * W, cudaMemcpyDeviceToHost));
    const int per = (int)((p->K_local + BP - 1) / BP);
    for (int b = 0; b < p->B; ++b) {
      const double* tb = tup.data() + (size_t)b * W;
      for (long long s = 0; s < p->K_local; ++s) {
        const size_t q = (size_t)b * p->K_local + s;
        const double mb = parts[((size_t)b * BP + s / per) * W];
        w[q] = (e[q] == 0.0 || !(tb[1] > 0.0)) ? 0.0 : e[q] * std::exp(-(mb - tb[0]) / p->cfg.lambda) / tb[1];
      }
    }
  });
}
int gpmppi_planner_flags(const gpmppi_planner* p, uint8_t* viol, uint8_t* coll, uint8_t* terminal,
                         uint8_t* alive) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    CK(cudaSetDevice(p->device));
    CK(cudaStreamSynchronize(p->stream));
    const long long S = p->slots();
    const size_t nw = (size_t)S * p->words;
    std::vector<uint32_t> vb(nw), cb(nw);
    CK(cudaMemcpy(vb.data(), p->d_viol, sizeof(uint32_t) * nw, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cb.data(), p->d_coll, sizeof(uint32_t) * nw, cudaMemcpyDeviceToHost));
    for (long long s = 0; s < S; ++s)
      for (int k = 0; k < p->T; ++k) {
        const size_t word = (size_t)s * p->words + (k >> 5);
        if (viol) viol[s * p->T + k] = (vb[word] >> (k & 31)) & 1u;
        if (coll) coll[s * p->T + k] = (cb[word] >> (k & 31)) & 1u;
      }
    if (terminal) CK(cudaMemcpy(terminal, p->d_term, S, cudaMemcpyDeviceToHost));
    if (alive) CK(cudaMemcpy(alive, p->d_alive, S, cudaMemcpyDeviceToHost));
  });
}

int gpmppi_planner_set_variance_path(gpmppi_planner* p, int path) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  if (path < 0 || path > 4) return fail(GPMPPI_INVALID_ARGUMENT, "unknown variance path");
  p->var_path = path;
  return GPMPPI_OK;
}
int gpmppi_planner_variance_path(const gpmppi_planner* p) { return p ? p->var_path : -1; }

int gpmppi_planner_bench_device(gpmppi_planner* p, const double* x0, const gpmppi_task* tasks,
                                int ticks, int flush_l2, double* tick_ms, double* phase_ms) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    CK(cudaSetDevice(p->device));
    if (ticks < 1) invalid("bench_device: ticks must be >= 1");
    if (p->K_local != p->K_total && !p->comm) invalid("bench_device: sharded planner without a communicator");
    stage_tick(p, x0, tasks);
    enqueue_h2d(p);
    void* flush = nullptr;
    size_t flush_bytes = 0;
    if (flush_l2) {
      int l2 = 0;
      CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, p->device));
      flush_bytes = (size_t)std::max(l2, 1 << 20) * 2;
      CK(cudaMalloc(&flush, flush_bytes));
    }
    // pass 1: per-phase events (an event between two kernels also breaks their
    // programmatic-dependent-launch overlap, so these sum to slightly more than a tick);
    // pass 2: the tick itself, one event pair around the unbroken kernel sequence
    std::vector<cudaEvent_t> evs((size_t)ticks * 7);
    for (auto& e : evs) CK(cudaEventCreate(&e));
    for (int t = 0; t < ticks; ++t) {
      cudaEvent_t* E = &evs[(size_t)t * 7];
      if (flush) CK(cudaMemsetAsync(flush, t & 0xff, flush_bytes, p->stream));  // outside the timed span
      enqueue_update(p, E);
      enqueue_tighten(p);
      CK(cudaEventRecord(E[4], p->stream));
      ++p->tick;  // the staged keys stay at the first tick: same work, fixed noise
    }
    for (int t = 0; t < ticks; ++t) {
      cudaEvent_t* E = &evs[(size_t)t * 7];
      if (flush) CK(cudaMemsetAsync(flush, (t + 7) & 0xff, flush_bytes, p->stream));
      CK(cudaEventRecord(E[5], p->stream));
      enqueue_update(p, nullptr);
      enqueue_tighten(p);
      CK(cudaEventRecord(E[6], p->stream));
      ++p->tick;
    }
    cudaError_t se = cudaStreamSynchronize(p->stream);
    if (flush) cudaFree(flush);
    CK(se);
    double ph[4] = {0, 0, 0, 0};
    for (int t = 0; t < ticks; ++t) {
      cudaEvent_t* E = &evs[(size_t)t * 7];
      for (int i = 0; i < 4; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, E[i], E[i + 1]));
        ph[i] += ms;
      }
      float tot = 0.f;
      CK(cudaEventElapsedTime(&tot, E[5], E[6]));
      if (tick_ms) tick_ms[t] = tot;
    }
    for (auto& e : evs) cudaEventDestroy(e);
    if (phase_ms)
      for (int i = 0; i < 4; ++i) phase_ms[i] = ph[i];  // rollout, variance, reduce+update, tightening
  });
}

int gpmppi_flush_l2(int device) {
  return guarded([&] {
    require_device(device);
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
    const size_t bytes = (size_t)std::max(l2, 1 << 20) * 2;
    // one flush buffer per device, kept for the process (an allocate/free per flush also
    // unmaps pages and cold-starts the TLBs, which is not what the flush is meant to model)
    static void* bufs[64] = {};
    if (device >= 64) invalid("flush_l2: device index too large");
    if (!bufs[device]) CK(cudaMalloc(&bufs[device], bytes));
    CK(cudaMemset(bufs[device], 0x5a, bytes));
    CK(cudaDeviceSynchronize());
  });
}

int gpmppi_planner_io_bytes(const gpmppi_planner* p, int64_t* h2d, int64_t* d2h) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  if (h2d) *h2d = (int64_t)p->B * (int64_t)(sizeof(gpm::TaskDev) + gpm::BatchStrides::X0 * sizeof(double));
  if (d2h) *d2h = (int64_t)p->B * (int64_t)(gpm::BatchStrides::OUT * sizeof(double) + sizeof(int));
  return GPMPPI_OK;
}

int gpmppi_debug_tc_profile(double* out16) {
  return guarded([&] { gpm::tc_profile_read(out16); });
}

int gpmppi_debug_tc_trace(double* out64) {
  return guarded([&] { gpm::tc_trace_read(out64); });
}

int gpmppi_debug_timeline(double* out32) {
  return guarded([&] { gpm::timeline_read(out32); });
}

int gpmppi_tuple_doubles(int horizon) { return gpm::tuple_doubles(horizon); }

int gpmppi_planner_set_shard(gpmppi_planner* p, int64_t begin, int64_t count) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    if (p->B != 1) invalid("set_shard: batched planners shard by robot, not by sample");
    if (begin < 0 || count < 1 || begin + count > p->K_total) invalid("set_shard: range outside [0, samples)");
    CK(cudaSetDevice(p->device));
    CK(cudaStreamSynchronize(p->stream));
    p->s_begin = begin;
    p->K_local = count;
    p->alloc_sample_buffers();  // frees the previous per-sample set, drops the tick graph
    CK(cudaStreamSynchronize(p->stream));
  });
}

int gpmppi_planner_plan_partial(gpmppi_planner* p, const double x0[5], const gpmppi_task* task,
                                void* device_tuple_out) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    CK(cudaSetDevice(p->device));
    if (p->B != 1) invalid("plan_partial: batched planner");
    if (p->noise_mode == gpm::NOISE_INJECTED && !p->injected_set) invalid("plan_partial: injected noise mode without noise");
    stage_tick(p, x0, task);
    enqueue_h2d(p);
    enqueue_samples(p, 0, nullptr);
    CK(cudaMemcpyAsync(device_tuple_out, p->d_rank_tuple, sizeof(double) * gpm::tuple_doubles(p->T),
                       cudaMemcpyDeviceToDevice, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  });
}

int gpmppi_planner_plan_finish(gpmppi_planner* p, const void* device_tuples, int n_ranks,
                               double command[2], gpmppi_diag* diag) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    const auto t0 = Clock::now();
    CK(cudaSetDevice(p->device));
    if (p->B != 1) invalid("plan_finish: batched planner");
    if (n_ranks < 1) invalid("plan_finish: n_ranks must be >= 1");
    check(gpm::launch_finish(static_cast<const double*>(device_tuples), n_ranks, p->T,
                             p->cfg.lambda, p->d_nom, p->cfg.lo, p->cfg.hi, p->d_out, p->K_total,
                             p->d_combined, p->stream),
          "finish kernel");
    copy_out_async(p);
    CK(cudaEventRecord(p->ev[0], p->stream));
    enqueue_tighten(p);
    CK(cudaMemcpyAsync(p->h_infeasible, p->d_infeasible, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
    CK(cudaEventSynchronize(p->ev[0]));
    const double t_cmd = ms_since(t0);
    CK(cudaStreamSynchronize(p->stream));
    fill_diag(p, command, diag, t_cmd, ms_since(t0));
    ++p->tick;
  });
}

// ---- reference free functions (mppi.hpp:60-79) on the device ----
}  // extern "C"
namespace {
struct DevBuf {  // scoped device allocation for the one-shot free functions
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { CK(cudaMalloc(&p, std::max<size_t>(bytes, 8))); }
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};
void h2d(void* d, const void* h, size_t bytes) { CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice)); }
void d2h(void* h, const void* d, size_t bytes) { CK(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost)); }
}  // namespace
extern "C" {

int gpmppi_rollout(const gpmppi_prediction_model* pm, const gpmppi_nominal* nominal,
                   const double* terrain_weights, int R, const double x0[5], const double* seq, int T,
                   int device, double* states, double* corrections) {
  return guarded([&] {  // mppi.cpp:80-111
    if (!pm || !nominal || !x0 || !seq || !states || !corrections) invalid("rollout: null argument");
    if (T < 0) invalid("rollout: negative horizon");
    if (pm->kind < 0 || pm->kind > 3) invalid("rollout: unknown prediction model");
    const bool gp = pm->kind == GPMPPI_MODEL_GP_ENSEMBLE;
    if (gp) {
      if (!pm->gp || pm->n_terrains < 1 || pm->gp->m != 2 * pm->n_terrains || R != pm->n_terrains)
        invalid("rollout: GP ensemble needs a model with 2M outputs and M weights");
      if (!terrain_weights || !on_simplex(terrain_weights, R, 1e-6))
        invalid("rollout: terrain weights must lie on the simplex");
      if (pm->gp->device != device) invalid("rollout: GP model lives on another device");
    }
    require_device(device);
    for (int i = 0; i < 5; ++i) states[i] = x0[i];
    if (T == 0) return;
    DevBuf dx(sizeof(double) * 5), ds(sizeof(double) * 2 * T), dw(sizeof(double) * std::max(R, 1)),
        dst(sizeof(double) * 5 * (T + 1)), dc(sizeof(double) * 4 * T);
    h2d(dx.p, x0, sizeof(double) * 5);
    h2d(ds.p, seq, sizeof(double) * 2 * T);
    if (gp) h2d(dw.p, terrain_weights, sizeof(double) * R);
    const gpm::NominalDev nom{nominal->tau_v, nominal->tau_omega, nominal->dt};
    const gpm::Edd5Dev edd{pm->edd5.alpha_l, pm->edd5.alpha_r, pm->edd5.x_icr, pm->edd5.y_icr_l,
                           pm->edd5.y_icr_r, pm->track_width};
    gpm::ModelDev M{};
    if (gp) M = pm->gp->dev;
    check(gpm::launch_rollout_one(M, pm->kind, nom, edd, dx.as<double>(), ds.as<double>(), T, dw.as<double>(),
                                  gp ? R : 0, dst.as<double>(), dc.as<double>(), 0),
          "rollout_one_kernel");
    CK(cudaDeviceSynchronize());
    d2h(states, dst.p, sizeof(double) * 5 * (T + 1));
    d2h(corrections, dc.p, sizeof(double) * 4 * T);
  });
}

int gpmppi_sample_perturbations(const gpmppi_mppi_config* cfg, uint64_t tick, int device, double* eps) {
  return guarded([&] {  // mppi.cpp:113-123 with the production (Philox) sampler
    if (!cfg || !eps) invalid("sample_perturbations: null argument");
    if (cfg->samples < 1 || cfg->horizon < 1) invalid("MppiConfig: samples and horizon must be >= 1");
    if (!(cfg->sigma_v2 > 0.0) || !(cfg->sigma_w2 > 0.0)) invalid("MppiConfig: sampling variances must be positive");
    require_device(device);
    const size_t cnt = (size_t)cfg->samples * cfg->horizon * 2;
    DevBuf d(sizeof(double) * cnt);
    check(gpm::launch_philox_noise(gpm::philox_key(cfg->seed, tick), 0, cfg->samples, cfg->horizon,
                                   std::sqrt(cfg->sigma_v2), std::sqrt(cfg->sigma_w2), d.as<double>(), 0),
          "philox_noise_kernel");
    CK(cudaDeviceSynchronize());
    d2h(eps, d.p, sizeof(double) * cnt);
  });
}

int gpmppi_trajectory_weights(const double* costs, int64_t K, double lambda, int device, double* w) {
  return guarded([&] {  // mppi.cpp:125-145
    if (!(lambda > 0.0)) invalid("trajectory_weights: lambda must be positive");
    if (K < 0 || (K > 0 && (!costs || !w))) invalid("trajectory_weights: bad arguments");
    if (K == 0) return;
    require_device(device);
    DevBuf dc(sizeof(double) * K), dw(sizeof(double) * K);
    h2d(dc.p, costs, sizeof(double) * K);
    check(gpm::launch_trajectory_weights(dc.as<double>(), K, lambda, dw.as<double>(), 0), "trajectory_weights_kernel");
    CK(cudaDeviceSynchronize());
    d2h(w, dw.p, sizeof(double) * K);
  });
}

int gpmppi_update_controls(const double* nominal, int T, const double* eps, const double* w, int64_t K,
                           const double lo[2], const double hi[2], int device, double* out) {
  return guarded([&] {  // mppi.cpp:147-164
    if (!nominal || !eps || !w || !lo || !hi || !out || T < 0 || K < 0)
      invalid("update_controls: one weight per sample required");
    if (T == 0) return;
    require_device(device);
    DevBuf dn(sizeof(double) * 2 * T), de(sizeof(double) * 2 * T * std::max<int64_t>(K, 1)),
        dw(sizeof(double) * std::max<int64_t>(K, 1)), dout(sizeof(double) * 2 * T);
    h2d(dn.p, nominal, sizeof(double) * 2 * T);
    if (K > 0) {
      h2d(de.p, eps, sizeof(double) * 2 * T * K);
      h2d(dw.p, w, sizeof(double) * K);
    }
    check(gpm::launch_update_controls(dn.as<double>(), T, de.as<double>(), dw.as<double>(), K, lo, hi,
                                      dout.as<double>(), 0),
          "update_controls_kernel");
    CK(cudaDeviceSynchronize());
    d2h(out, dout.p, sizeof(double) * 2 * T);
  });
}

int gpmppi_shift_horizon(const double* seq, int T, int device, double* out) {
  return guarded([&] {  // mppi.cpp:166-173
    if (T < 1) invalid("shift_horizon: empty sequence");
    if (!seq || !out) invalid("shift_horizon: null argument");
    require_device(device);
    DevBuf ds(sizeof(double) * 2 * T), dout(sizeof(double) * 2 * T);
    h2d(ds.p, seq, sizeof(double) * 2 * T);
    check(gpm::launch_shift_horizon(ds.as<double>(), T, dout.as<double>(), 0), "shift_horizon_kernel");
    CK(cudaDeviceSynchronize());
    d2h(out, dout.p, sizeof(double) * 2 * T);
  });
}

int gpmppi_nccl_unique_id(void* out) {
  if (!out) return fail(GPMPPI_INVALID_ARGUMENT, "nccl_unique_id: null output");
  return guarded([&] {
    ncclUniqueId id;
    nccl_check(nccl_required().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
  });
}

int gpmppi_planner_attach_comm(gpmppi_planner* p, const void* unique_id, int n_ranks, int rank) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    if (!unique_id) invalid("attach_comm: null unique id");
    if (p->B != 1) invalid("attach_comm: batched planners shard by robot, not by sample");
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) invalid("attach_comm: bad rank / world size");
    if (p->comm) invalid("attach_comm: a communicator is already attached");
    if (p->K_total < n_ranks) invalid("attach_comm: fewer samples than ranks");
    const NcclApi& api = nccl_required();
    CK(cudaSetDevice(p->device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    ncclComm_t c = nullptr;
    nccl_check(api.comm_init_rank(&c, n_ranks, id, rank), "ncclCommInitRank");  // collective
    // contiguous global sample range of this rank (gpmppi.shard_range)
    const long long base = p->K_total / n_ranks, extra = p->K_total % n_ranks;
    p->s_begin = (long long)rank * base + std::min<long long>(rank, extra);
    p->K_local = base + (rank < extra ? 1 : 0);
    p->alloc_sample_buffers();  // drops any captured tick graph
    p->d_gathered = p->dalloc<double>((size_t)n_ranks * gpm::tuple_doubles(p->T));
    p->comm = c;
    p->n_ranks = n_ranks;
    p->rank = rank;
    CK(cudaStreamSynchronize(p->stream));
  });
}

int gpmppi_planner_shard(const gpmppi_planner* p, int64_t* begin, int64_t* count, int* n_ranks, int* rank) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  if (begin) *begin = p->s_begin;
  if (count) *count = p->K_local;
  if (n_ranks) *n_ranks = p->n_ranks;
  if (rank) *rank = p->rank;
  return GPMPPI_OK;
}

int gpmppi_planner_set_command_first(gpmppi_planner* p, int on) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    finish_pending(p, nullptr);
    p->command_first = on != 0;
  });
}

int gpmppi_planner_wait_tightening(gpmppi_planner* p, gpmppi_diag* diag) {
  if (!p) return fail(GPMPPI_INVALID_ARGUMENT, "null planner");
  return guarded([&] {
    CK(cudaSetDevice(p->device));
    const bool had = p->tightening_pending;
    finish_pending(p, diag);
    if (!had && diag)  // nothing pending: the last tick's completed diagnostics, if any
      for (int b = 0; b < (int)p->pending_diag.size(); ++b) diag[b] = p->pending_diag[b];
  });
}

// select_kernel_grid (gp.cpp:274-366): base lengthscales and pooled output variance on the
// host, every cell's Cholesky + LML on the device (fit.cu), the reference's sweep order and
// first-strictly-greater argmax across both passes on the host.
int gpmppi_select_kernel_grid(const double* inputs, const double* outputs, int64_t n64, int64_t m64, int device,
                              double kernel6[6], double* best_lml) {
  return guarded([&] {
    if (!inputs || !outputs || !kernel6) invalid("select_kernel_grid: null argument");
    if (n64 < 2) invalid("select_kernel_grid: need at least 2 points");
    if (m64 < 1) invalid("select_kernel_grid: outputs must be n x m with m >= 1");
    if (n64 > 8192) invalid("select_kernel_grid: n too large for the device grid");
    const int n = (int)n64, m = (int)m64;
    require_device(device);
    double base[4];
    for (int d = 0; d < 4; ++d) {  // gp.cpp:281-285
      double mu = 0.0;
      for (int i = 0; i < n; ++i) mu += inputs[(size_t)i * 4 + d];
      mu /= n;
      double var = 0.0;
      for (int i = 0; i < n; ++i) var += (inputs[(size_t)i * 4 + d] - mu) * (inputs[(size_t)i * 4 + d] - mu);
      base[d] = std::max(std::sqrt(var / (double)(n - 1)), 1e-3);
    }
    double pooled = 0.0;  // gp.cpp:286-291
    for (int j = 0; j < m; ++j) {
      double mu = 0.0;
      for (int i = 0; i < n; ++i) mu += outputs[(size_t)i * m + j];
      mu /= n;
      double v = 0.0;
      for (int i = 0; i < n; ++i) v += (outputs[(size_t)i * m + j] - mu) * (outputs[(size_t)i * m + j] - mu);
      pooled += v / (double)(n - 1);
    }
    pooled = std::max(pooled / (double)m, 1e-10);
    std::vector<double> sc((size_t)n * 4), sq(n), d2((size_t)n * n);  // gp.cpp:294-299
    for (int i = 0; i < n; ++i) {
      double q = 0.0;
      for (int d = 0; d < 4; ++d) {
        sc[(size_t)i * 4 + d] = inputs[(size_t)i * 4 + d] / base[d];
        q += sc[(size_t)i * 4 + d] * sc[(size_t)i * 4 + d];
      }
      sq[i] = q;
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double dot = 0.0;
        for (int d = 0; d < 4; ++d) dot += sc[(size_t)i * 4 + d] * sc[(size_t)j * 4 + d];
        d2[(size_t)i * n + j] = -2.0 * dot + sq[i] + sq[j];
      }
    for (int i = 0; i < n; ++i)
      for (int j = i; j < n; ++j) {
        const double v = std::max(0.5 * (d2[(size_t)i * n + j] + d2[(size_t)j * n + i]), 0.0);
        d2[(size_t)i * n + j] = d2[(size_t)j * n + i] = v;
      }
    auto logspace = [](double lo, double hi, int k) {
      std::vector<double> v(k);
      for (int i = 0; i < k; ++i) v[i] = std::pow(10.0, lo + (hi - lo) * (k == 1 ? 0.0 : (double)i / (k - 1)));
      return v;
    };
    double best = -std::numeric_limits<double>::infinity();
    double best_sv = pooled, best_s = 1.0, best_nv = pooled * 0.1;
    auto sweep = [&](const std::vector<double>& svs, const std::vector<double>& ss, const std::vector<double>& nvs) {
      std::vector<double> cells;
      for (double sv : svs)
        for (double s : ss)
          for (double nv : nvs) {
            cells.push_back(sv);
            cells.push_back(s);
            cells.push_back(nv);
          }
      const int nc = (int)(cells.size() / 3);
      std::vector<double> scores(nc);
      CK(gpm::device_lml_grid(d2.data(), outputs, n, m, cells.data(), nc, scores.data()));
      for (int c = 0; c < nc; ++c)  // sweep order, strictly greater (gp.cpp:331-340)
        if (scores[c] > best) {
          best = scores[c];
          best_sv = cells[3 * c];
          best_s = cells[3 * c + 1];
          best_nv = cells[3 * c + 2];
        }
    };
    {
      std::vector<double> svs, nvs;
      for (double f : logspace(-1.5, 1.5, 5)) svs.push_back(pooled * f);
      for (double f : logspace(-3.0, 0.5, 5)) nvs.push_back(pooled * f);
      sweep(svs, logspace(-1.0, 1.0, 7), nvs);
    }
    {
      const double sv0 = best_sv, s0 = best_s, nv0 = best_nv;
      std::vector<double> svs, ss, nvs;
      for (double f : logspace(-0.5, 0.5, 5)) svs.push_back(sv0 * f);
      for (double f : logspace(-0.35, 0.35, 7)) ss.push_back(s0 * f);
      for (double f : logspace(-0.6, 0.6, 5)) nvs.push_back(nv0 * f);
      sweep(svs, ss, nvs);
    }
    kernel6[0] = best_sv;
    for (int d = 0; d < 4; ++d) kernel6[1 + d] = base[d] * best_s;
    kernel6[5] = best_nv;
    if (best_lml) *best_lml = best;
  });
}

int gpmppi_combine_tuples_host(const double* tuples, int n_ranks, int horizon, double lambda,
                               double* out) {
  if (!tuples || !out || n_ranks < 1 || horizon < 1 || !(lambda > 0.0))
    return fail(GPMPPI_INVALID_ARGUMENT, "combine_tuples: bad arguments");
  gpm::combine_tuples(tuples, n_ranks, horizon, lambda, out);
  return GPMPPI_OK;
}

}  // extern "C"
