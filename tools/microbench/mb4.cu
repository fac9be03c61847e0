// Microbenchmark 4: issue model of DFMA mixed with ALU/FMA-pipe instructions
// on sm_100a. Each variant runs 16 independent fp64 accumulator chains per
// thread; per "genotype" it executes 1 DFMA plus X extra integer ops.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__global__ void kern(int iters, uint32_t seed, double c, double* out) {
  double acc[16];
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = seed * (threadIdx.x + 7 * i + 1);
  double cc = c + threadIdx.x;  // coefficient in a regular register
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double d;
      if (V == 0) {  // DFMA, operand pair from registers computed once (no extra op)
        d = __hiloint2double(0, (int)w[k & 3]);
      } else if (V == 1) {  // LOP3 + (maybe MOV) + DFMA
        d = __hiloint2double(0, (int)(w[k & 3] & (3u << (2 * k))));
      } else if (V == 2) {  // IADD-based extraction (ALU), same count
        d = __hiloint2double((int)(w[k & 3] & (3u << (2 * k))), 0x3ff00000 ^ 0x3ff00000);
      } else {  // LOP3 into the hi word with a constant exponent (normal numbers)
        d = __hiloint2double((int)((w[k & 3] & (3u << (2 * (k & 7)))) | 0x3ff00000), 0);
      }
      acc[k] = fma(d, cc, acc[k]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = w[i] * 1664525u + 1013904223u;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run(const char* name, int sms, int clk, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000, bs = 256, grid = sms * 8;
  kern<V><<<grid, bs>>>(iters, 2654435761u, 1.5, out);
  cudaEventRecord(e0);
  kern<V><<<grid, bs>>>(iters, 2654435761u, 1.5, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double g = (double)grid * bs * iters * 16;
  printf("%-36s %.2f DFMA/clk/SM at rated clock\n", name, g / (ms * 1e-3) / sms / (clk * 1e3));
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, (size_t)sms * 8 * 256 * 8);
  for (int r = 0; r < 2; ++r) {
    run<0>("dfma (reg operands, 0 extra)", sms, clk, out);
    run<1>("lop3 + dfma (denormal lo)", sms, clk, out);
    run<2>("lop3 + dfma (hi field, lo 0)", sms, clk, out);
    run<3>("lop3|exp + dfma (normal hi)", sms, clk, out);
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
