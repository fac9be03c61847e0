// Microbenchmark 2: the "denormal-injection" decode. Each 2-bit dosage field
// of a packed word is masked in place (LOP3) and used directly as the low
// word of an fp64 operand with zero high word (a denormal r*2^(2k-1074));
// one DFMA per genotype accumulates it against a pre-scaled coefficient.
// Measures genotypes/clk/SM with data in registers (no memory traffic).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double fld(uint32_t w, int k) {
  return __hiloint2double(0, (int)(w & (3u << (2 * k))));
}

__global__ void decode_fma(int iters, const uint32_t* __restrict__ seedw, double* out) {
  uint32_t w0 = seedw[threadIdx.x & 63], w1 = w0 * 2654435761u, w2 = w1 ^ 0x9e3779b9u, w3 = w2 * 7u;
  double c0 = 1e300, c1 = 2e300, c2 = 3e300, c3 = 4e300;
  double acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      acc[k] = fma(fld(w0, k), c0, acc[k]);
      acc[k] = fma(fld(w1, k), c1, acc[k]);
      acc[k] = fma(fld(w2, k), c2, acc[k]);
      acc[k] = fma(fld(w3, k), c3, acc[k]);
    }
    w0 += 0x01010101u; w1 ^= w0; w2 += w1; w3 ^= w2;  // keep the words live
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* sw; double* out;
  cudaMalloc(&sw, 64 * 4); cudaMalloc(&out, (size_t)sms * 2048 * 8);
  uint32_t h[64]; for (int i = 0; i < 64; ++i) h[i] = 0x9e3779b9u * (i + 1);
  cudaMemcpy(sw, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  for (int bs : {128, 256, 512}) for (int per : {2, 4, 8}) {
    int grid = sms * per;
    if (bs * per > 2048) continue;
    decode_fma<<<grid, bs>>>(iters, sw, out);
    cudaEventRecord(e0);
    decode_fma<<<grid, bs>>>(iters, sw, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double g = (double)grid * bs * iters * 64;
    printf("decode_fma bs=%d blocks/SM=%d: %.2f genotypes/clk/SM at rated clock (%.1f Ggeno/s, eq %.0f GB/s packed)\n",
           bs, per, g / (ms * 1e-3) / sms / (clk * 1e3), g / (ms * 1e6), g / 4 / (ms * 1e6));
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
