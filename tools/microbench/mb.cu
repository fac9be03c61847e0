// Microbenchmarks that decide the packed-genotype kernel design on sm_100a:
//  (1) streaming read bandwidth with 128-bit loads (the HBM roofline we can reach),
//  (2) LDS.64 lookups into a 16-entry fp64 table (warp-uniform table, per-lane
//      4-bit index) vs 32 distinct addresses, in lookups/clk/SM,
//  (3) DADD throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void stream_read(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride),
          d = __ldcs(p + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n; i += stride) { uint4 a = p[i]; acc ^= a.x ^ a.y ^ a.z ^ a.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

// mode 0: 16-entry table, per-lane random nibble (<=16 distinct addresses).
// mode 1: 32 distinct addresses (lane-private slot).
template <int MODE>
__global__ void lds_lookup(int iters, double* out, uint32_t seed) {
  __shared__ double tab[8][32];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) (&tab[0][0])[i] = i * 0.5;
  __syncthreads();
  uint32_t x = seed ^ (threadIdx.x * 2654435761u);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t w = x;
#pragma unroll
    for (int k = 0; k < 8; k += 4) {
      int i0, i1, i2, i3;
      if (MODE == 0) {
        i0 = (w >> (4 * k)) & 15; i1 = (w >> (4 * k + 4)) & 15;
        i2 = (w >> (4 * k + 8)) & 15; i3 = (w >> (4 * k + 12)) & 15;
      } else {
        i0 = lane; i1 = lane; i2 = lane; i3 = lane;
      }
      a0 += tab[k][i0]; a1 += tab[k + 1][i1]; a2 += tab[k + 2][i2]; a3 += tab[k + 3][i3];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

__global__ void dadd_rate(int iters, double* out) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  const double b = 1.0000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = a[k] + b;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("SMs %d clockRate %d kHz\n", sms, clk);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;

  // (1) streaming read: 4 GiB
  size_t bytes = (size_t)4 << 30;
  uint4* buf; uint32_t* o;
  CK(cudaMalloc(&buf, bytes)); CK(cudaMalloc(&o, 64));
  CK(cudaMemset(buf, 1, bytes));
  for (int bs : {256, 512}) for (int per : {4, 8, 16}) {
    int grid = sms * per;
    stream_read<<<grid, bs>>>(buf, bytes / 16, o);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) stream_read<<<grid, bs>>>(buf, bytes / 16, o);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("stream_read bs=%d grid=%d : %.1f GB/s\n", bs, grid, 5.0 * bytes / (ms * 1e6));
  }
  CK(cudaFree(buf));

  double* out; CK(cudaMalloc(&out, (size_t)sms * 32 * 1024 * 8));
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode) for (int bs : {256, 512, 1024}) {
    int grid = sms * (2048 / bs);
    auto launch = [&]() {
      if (mode == 0) lds_lookup<0><<<grid, bs>>>(iters, out, 7);
      else lds_lookup<1><<<grid, bs>>>(iters, out, 7);
    };
    launch();
    CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double lookups = (double)grid * bs * iters * 8;
    double per_clk_sm = lookups / (ms * 1e-3) / sms / (clk * 1e3);
    printf("lds mode=%d bs=%d: %.2f lookups/clk/SM (at rated clock), %.3f ms\n", mode, bs, per_clk_sm, ms);
  }
  {
    int bs = 512, grid = sms * 4;
    dadd_rate<<<grid, bs>>>(iters, out);
    CK(cudaEventRecord(e0)); dadd_rate<<<grid, bs>>>(iters, out); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double ops = (double)grid * bs * iters * 8;
    printf("dadd: %.2f /clk/SM (at rated clock)\n", ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
