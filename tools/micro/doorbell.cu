// Host round-trip latency of one "tick" trigger: (a) cudaGraphLaunch of a graph with an
// H2D copy node and a chain of PDL kernels, the last one publishing a sequence number into
// mapped pinned memory that the host polls; (b) the same chain pre-launched behind a
// doorbell kernel that polls a mapped host word (the host writes the input block and the
// doorbell, then polls the completion word). Prints median / p99 microseconds.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o doorbell doorbell.cu
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s failed: %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// one link of the chain: every block reads the staged input, the last kernel publishes
__global__ void link_kernel(const double* in, double* scratch, volatile double* done, int last) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) scratch[blockIdx.x] = in[0] + in[7] * 1e-9;
  if (last && blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    done[0] = in[7];
  }
}

// waits for the host's doorbell (mapped word), then copies the mapped input block
__global__ void bell_kernel(const volatile double* bell, const double* h_in, double* d_in, int words,
                            double* expect) {
  pdl_trigger();
  __shared__ double seen;
  if (threadIdx.x == 0) {
    const double want = expect[0] + 1.0;
    double v;
    do {
      v = bell[0];
    } while (v < want);
    expect[0] = v;
    seen = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < words; i += blockDim.x) d_in[i] = ((const volatile double*)h_in)[i];
  (void)seen;
}

// copies the mapped (host) input block into device memory: the first node instead of a copy
__global__ void stage_kernel(const double* h_in, double* d_in, int words) {
  pdl_trigger();
  for (int i = threadIdx.x; i < words; i += blockDim.x) d_in[i] = ((const volatile double*)h_in)[i];
}

template <class... KArgs, class... Args>
cudaError_t launch(void (*k)(KArgs...), int grid, int block, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(grid);
  c.blockDim = dim3(block);
  c.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = at;
  c.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&c, k, args...);
}

static void stats(const char* name, std::vector<double>& v) {
  std::sort(v.begin(), v.end());
  printf("%-44s median %7.2f us  p99 %7.2f us\n", name, v[v.size() / 2], v[(size_t)(v.size() * 0.99)]);
}

int main() {
  const int words = 512, chain = 6, iters = 2000;
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double *h_in, *h_done, *h_bell, *dh_in, *dh_done, *dh_bell, *d_in, *d_scr, *d_expect;
  CK(cudaHostAlloc(&h_in, words * 8, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_done, 64, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_bell, 64, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&dh_in, h_in, 0));
  CK(cudaHostGetDevicePointer((void**)&dh_done, h_done, 0));
  CK(cudaHostGetDevicePointer((void**)&dh_bell, h_bell, 0));
  CK(cudaMalloc(&d_in, words * 8));
  CK(cudaMalloc(&d_scr, 4096 * 8));
  CK(cudaMalloc(&d_expect, 8));
  CK(cudaMemset(d_expect, 0, 8));
  for (int i = 0; i < words; ++i) h_in[i] = i;
  h_done[0] = 0;
  h_bell[0] = 0;
  using Clk = std::chrono::steady_clock;
  auto spin = [&](double want) {
    while (((volatile double*)h_done)[0] != want) {
    }
  };
  // (a) graph: H2D node + chain
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  CK(cudaMemcpyAsync(d_in, h_in, words * 8, cudaMemcpyHostToDevice, st));
  for (int k = 0; k < chain; ++k)
    CK(launch(link_kernel, 148, 256, st, k > 0, (const double*)d_in, d_scr, dh_done, k == chain - 1 ? 1 : 0));
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  std::vector<double> ta;
  double seq = 0;
  for (int it = 0; it < iters; ++it) {
    seq += 1;
    const auto t0 = Clk::now();
    h_in[7] = seq;
    CK(cudaGraphLaunch(ge, st));
    spin(seq);
    ta.push_back(std::chrono::duration<double, std::micro>(Clk::now() - t0).count());
  }
  CK(cudaStreamSynchronize(st));
  // (b) doorbell graph: bell kernel + chain (PDL from the bell kernel); launched one tick ahead
  cudaGraph_t gb;
  cudaGraphExec_t gbe;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  CK(launch(bell_kernel, 1, 256, st, false, (const volatile double*)dh_bell, (const double*)dh_in, d_in, words,
            d_expect));
  for (int k = 0; k < chain; ++k)
    CK(launch(link_kernel, 148, 256, st, true, (const double*)d_in, d_scr, dh_done, k == chain - 1 ? 1 : 0));
  CK(cudaStreamEndCapture(st, &gb));
  CK(cudaGraphInstantiate(&gbe, gb, 0));
  CK(cudaMemcpy(d_expect, &seq, 8, cudaMemcpyHostToDevice));
  h_bell[0] = seq;
  std::vector<double> tb;
  CK(cudaGraphLaunch(gbe, st));  // armed for seq + 1
  for (int it = 0; it < iters; ++it) {
    seq += 1;
    const auto t0 = Clk::now();
    h_in[7] = seq;
    ((volatile double*)h_bell)[0] = seq;
    spin(seq);
    const double us = std::chrono::duration<double, std::micro>(Clk::now() - t0).count();
    tb.push_back(us);
    if (it + 1 < iters) CK(cudaGraphLaunch(gbe, st));  // arm the next tick (outside the timed span)
  }
  CK(cudaStreamSynchronize(st));
  // (c) graph: a staging kernel reading the mapped input block (no copy node) + chain
  cudaGraph_t gc;
  cudaGraphExec_t gce;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  CK(launch(stage_kernel, 1, 256, st, false, (const double*)dh_in, d_in, words));
  for (int k = 0; k < chain; ++k)
    CK(launch(link_kernel, 148, 256, st, true, (const double*)d_in, d_scr, dh_done, k == chain - 1 ? 1 : 0));
  CK(cudaStreamEndCapture(st, &gc));
  CK(cudaGraphInstantiate(&gce, gc, 0));
  std::vector<double> tc;
  for (int it = 0; it < iters; ++it) {
    seq += 1;
    const auto t0 = Clk::now();
    h_in[7] = seq;
    CK(cudaGraphLaunch(gce, st));
    spin(seq);
    tc.push_back(std::chrono::duration<double, std::micro>(Clk::now() - t0).count());
  }
  CK(cudaStreamSynchronize(st));
  // (d) graph: the chain alone (input already on the device: the launch-path floor)
  cudaGraph_t gd;
  cudaGraphExec_t gde;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < chain; ++k)
    CK(launch(link_kernel, 148, 256, st, k > 0, (const double*)dh_in, d_scr, dh_done, k == chain - 1 ? 1 : 0));
  CK(cudaStreamEndCapture(st, &gd));
  CK(cudaGraphInstantiate(&gde, gd, 0));
  std::vector<double> td;
  for (int it = 0; it < iters; ++it) {
    seq += 1;
    const auto t0 = Clk::now();
    h_in[7] = seq;
    CK(cudaGraphLaunch(gde, st));
    spin(seq);
    td.push_back(std::chrono::duration<double, std::micro>(Clk::now() - t0).count());
  }
  CK(cudaStreamSynchronize(st));
  stats("graph launch (H2D node + 6 PDL kernels)", ta);
  stats("graph launch (staging kernel + 6 PDL kernels)", tc);
  stats("graph launch (6 PDL kernels, mapped input)", td);
  stats("pre-launched doorbell (+ 6 PDL kernels)", tb);
  return 0;
}
