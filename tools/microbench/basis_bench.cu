// Times the Krylov-basis kernels (basis_kernels.cu) at the Lanczos sizes:
// per-call device time of back-to-back launches (CUDA events), including the
// reduction finalize. Build: make -C tools/microbench ; run on the GPU box.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "../../paper_1808_03374_b200/csrc/kernels.hpp"

using namespace gkb::dev;

// Device time per call: `iters` calls captured into one CUDA graph (no host
// launch overhead in the measurement), replayed 5 times.
template <class F>
static double time_us(F&& f, int iters, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < iters; ++i) f();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(a, s);
  for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return 1e3 * ms / (5.0 * iters);
}

// Host cost of one launch call (wall clock, stream never drained in between)
template <class F>
static double host_us(F&& f, int iters, cudaStream_t s) {
  cudaStreamSynchronize(s);
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) f();
  const auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  RedScratch rs{};
  rs.cap = 1 << 20;
  cudaMalloc(&rs.partial, sizeof(double) * rs.cap);
  cudaMemset(rs.partial, 0, sizeof(double) * rs.cap);
  init_red_scratch(rs);
  const int64_t lens[] = {10000, 100000, 500000};
  const int64_t cols[] = {1, 25, 50};
  double *Q, *v, *c, *out, *W, *D;
  const int64_t maxlen = 500000, maxc = 64;
  cudaMalloc(&Q, sizeof(double) * maxlen * maxc);
  cudaMalloc(&D, sizeof(double) * maxlen * maxc);
  cudaMalloc(&v, sizeof(double) * maxlen);
  cudaMalloc(&c, sizeof(double) * 4096);
  cudaMalloc(&out, sizeof(double) * 4096);
  cudaMalloc(&W, sizeof(double) * maxc * maxc);
  std::vector<double> h(maxlen * maxc);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-3 * (double)((i * 2654435761u) % 2001) - 1.0;
  cudaMemcpy(Q, h.data(), sizeof(double) * maxlen * maxc, cudaMemcpyHostToDevice);
  cudaMemcpy(v, h.data(), sizeof(double) * maxlen, cudaMemcpyHostToDevice);
  cudaMemcpy(c, h.data(), sizeof(double) * 4096, cudaMemcpyHostToDevice);
  cudaMemcpy(W, h.data(), sizeof(double) * maxc * maxc, cudaMemcpyHostToDevice);
  printf("host launch cost: div_copy %.2f us, dot %.2f us\n",
         host_us([&] { div_copy(v, 1.0, D, 10000, s); }, 2000, s),
         host_us([&] { dot(Q, v, 10000, rs, out, s); }, 2000, s));
  for (int64_t len : lens) {
    printf("len %lld\n", (long long)len);
    printf("  dot              %7.2f us\n", time_us([&] { dot(Q, v, len, rs, out, s); }, 200, s));
    printf("  axpy_norms       %7.2f us\n",
           time_us([&] { axpy_norms(1e-9, Q, v, len, rs, out, s); }, 200, s));
    printf("  axpy_dev         %7.2f us\n", time_us([&] { axpy_dev(c, Q, v, len, s); }, 200, s));
    printf("  div_copy         %7.2f us\n", time_us([&] { div_copy(v, 1.0, D, len, s); }, 200, s));
    for (int64_t nc : cols) {
      const double bytes = 8.0 * len * (nc + 1);
      const double tt = time_us([&] { gemv_t(Q, len, len, nc, v, true, rs, out, s); }, 200, s);
      const double tn =
          time_us([&] { gemv_n(Q, len, len, nc, c, v, 1.0, -1e-12, true, rs, out, s); }, 200, s);
      printf("  ncols %3lld  gemv_t %7.2f us (%6.0f GB/s)  gemv_n %7.2f us (%6.0f GB/s)\n",
             (long long)nc, tt, bytes / tt * 1e-3, tn, (bytes + 8.0 * len) / tn * 1e-3);
    }
    const double tg = time_us([&] { gemm_small(Q, len, len, 50, W, 50, 25, D, len, s); }, 50, s);
    printf("  gemm_small 50->25 %7.2f us (%6.0f GB/s)\n", tg, 8.0 * len * 75 / tg * 1e-3);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
