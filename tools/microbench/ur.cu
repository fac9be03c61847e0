// Does a warp-uniform coefficient loaded from shared memory reach DFMA as a
// uniform-register operand? Variants: plain LDS, __shfl_sync broadcast,
// constant-bank (__constant__) load with a uniform index.
#include <cstdint>

__constant__ double c_coef[4096];

__device__ __forceinline__ double fld(uint32_t w, int k) {
  return __hiloint2double(0, (int)(w & (3u << (2 * k))));
}

template <int V>
__global__ void k(const uint4* __restrict__ src, const double* __restrict__ gcoef, int nq, double* out) {
  __shared__ double cs[4096];
  for (int t = threadIdx.x; t < 4096; t += blockDim.x) cs[t] = gcoef[t];
  __syncthreads();
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int q = 0; q < nq; ++q) {
    const uint4 c = src[q * 1024 + threadIdx.x];
    double ca;
    if (V == 0) ca = cs[4 * q];
    else if (V == 1) ca = __shfl_sync(0xffffffffu, cs[4 * q], 0);
    else ca = c_coef[4 * q];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(fld(c.x, i), ca, acc[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[threadIdx.x] = s;
}
template __global__ void k<0>(const uint4*, const double*, int, double*);
template __global__ void k<1>(const uint4*, const double*, int, double*);
template __global__ void k<2>(const uint4*, const double*, int, double*);
