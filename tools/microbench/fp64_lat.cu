// Dependent-chain latency of FP64 DADD / DMUL / DFMA and FP32 FADD on one warp
// (clock64 around 1024 chained ops), to size sequential fp64 recurrences.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double x, float xf, long long* out, double* sink, float* sinkf) {
  double a = x, b = x * 0.5;
  float af = xf;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) a = __dmul_rn(a, 0.999999);
  long long t2 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) a = __fma_rn(a, 0.999999, b);
  long long t3 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) af = __fadd_rn(af, 1.0f);
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3;
  }
  sink[threadIdx.x] = a;
  sinkf[threadIdx.x] = af;
}

int main() {
  long long* o; double* s; float* sf;
  cudaMalloc(&o, 64); cudaMalloc(&s, 1024); cudaMalloc(&sf, 512);
  for (int rep = 0; rep < 2; ++rep) k_lat<<<1, 32>>>(1.0, 1.0f, o, s, sf);
  long long h[4];
  cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: DADD %.1f DMUL %.1f DFMA %.1f FADD %.1f\n", h[0] / 1024.0,
         h[1] / 1024.0, h[2] / 1024.0, h[3] / 1024.0);
  return 0;
}
