// Microbenchmarks for the fixed-point tensor-core GEMV design:
//  (1) mma.sync.m16n8k32 u8 x s8 -> s32 issue rate on sm_100a (MMAs/clk/SM),
//  (2) a prototype of the packed GEMV main loop: stream a 2-bit tile layout
//      (16 rows x 128 cols = 512 B per tile, fragment order), expand each 32-bit
//      word into four int8 fragment registers, 4 MMAs per 16-byte load against
//      B fragments (coefficient digits) from shared memory. Reports GB/s of
//      packed bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma mma.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);           \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CHAINS>
__global__ void mma_rate(int iters, int* out, long long* cyc) {
  int acc[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[c][i] = 0;
  uint32_t a = 0x01020102u ^ threadIdx.x, b = 0x7f81017fu ^ (threadIdx.x << 3);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) mma_u8s8(acc[c], a, a ^ c, a + c, a, b, b ^ c);
  }
  __syncthreads();
  long long t1 = clock64();
  int s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Prototype GEMV main loop. Layout: strip r (16 rows) x tiles kt, tile = 512 B,
// thread t of the warp reads uint4 #t of the tile. CTA = 8 warps (8 strips)
// x KT_CTA tiles of K; digits for the CTA's K range in shared memory
// (16 B per (word-col, digit)).
// MODE 0: as described; 1: no MMA (expansion xor-folded); 2: two accumulator
// chains (alternating MMAs); 3: B fragments from registers (no LDS)
template <int DEPTH, int MINB, int MODE = 0>
__global__ void __launch_bounds__(256, MINB) gemv_proto(const uint4* __restrict__ lay, int64_t KT,
                                                  int kt_cta, const uint4* __restrict__ digits,
                                                  double* __restrict__ out) {
  extern __shared__ uint4 dg[];  // kt_cta * 8 word-cols * 8 digits
  const int ktiles = kt_cta;
  const int64_t kt0 = (int64_t)blockIdx.y * kt_cta;
  for (int i = threadIdx.x; i < ktiles * 64; i += 256) dg[i] = digits[kt0 * 64 + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tid = lane & 3;
  const int64_t strip = (int64_t)blockIdx.x * 8 + warp;
  const uint4* src = lay + (strip * KT + kt0) * 32 + lane;
  int acc[4] = {0, 0, 0, 0};
  int acc2[4] = {0, 0, 0, 0};
  uint32_t xf = 0;
  uint4 buf[DEPTH];
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) buf[d] = d < ktiles ? __ldcs(src + d * 32) : make_uint4(0, 0, 0, 0);
  for (int kt = 0; kt < ktiles; kt += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const uint4 w = buf[d];
      if (kt + d + DEPTH < ktiles) buf[d] = __ldcs(src + (kt + d + DEPTH) * 32);
      if (kt + d < ktiles) {
        uint4 b01, b23;
        if (MODE == 3) {
          b01 = make_uint4(lane, lane * 3, lane * 5, lane * 7);
          b23 = make_uint4(lane * 11, lane * 13, lane * 17, lane * 19);
        } else {
          b01 = dg[((kt + d) * 8 + tid) * 8 + g];
          b23 = dg[((kt + d) * 8 + tid + 4) * 8 + g];
        }
        const uint32_t m = 0x03030303u;
        if (MODE == 1) {
          xf ^= (w.x & m) ^ (w.y & m) ^ ((w.x >> 2) & m) ^ ((w.y >> 2) & m) ^ b01.x ^ b23.w;
          xf ^= ((w.z >> 4) & m) ^ ((w.w >> 4) & m) ^ ((w.z >> 6) & m) ^ ((w.w >> 6) & m);
        } else if (MODE == 2) {
          mma_u8s8(acc, w.x & m, w.y & m, (w.x >> 2) & m, (w.y >> 2) & m, b01.x, b01.y);
          mma_u8s8(acc2, (w.x >> 4) & m, (w.y >> 4) & m, (w.x >> 6) & m, (w.y >> 6) & m, b01.z, b01.w);
          mma_u8s8(acc, w.z & m, w.w & m, (w.z >> 2) & m, (w.w >> 2) & m, b23.x, b23.y);
          mma_u8s8(acc2, (w.z >> 4) & m, (w.w >> 4) & m, (w.z >> 6) & m, (w.w >> 6) & m, b23.z, b23.w);
        } else {
          mma_u8s8(acc, w.x & m, w.y & m, (w.x >> 2) & m, (w.y >> 2) & m, b01.x, b01.y);
          mma_u8s8(acc, (w.x >> 4) & m, (w.y >> 4) & m, (w.x >> 6) & m, (w.y >> 6) & m, b01.z, b01.w);
          mma_u8s8(acc, w.z & m, w.w & m, (w.z >> 2) & m, (w.w >> 2) & m, b23.x, b23.y);
          mma_u8s8(acc, (w.z >> 4) & m, (w.w >> 4) & m, (w.z >> 6) & m, (w.w >> 6) & m, b23.z, b23.w);
        }
      }
    }
  }
  double v = (double)acc[0] + 256.0 * acc[1] + (double)acc[2] * 3.0 + acc[3] + acc2[0] + acc2[3] + xf;
  out[(strip * gridDim.y + blockIdx.y) * 32 + lane] = v;
}

// R row strips per warp share each B fragment (LDS amortized R times).
template <int R, int DEPTH, int MINB>
__global__ void __launch_bounds__(256, MINB) gemv_multi(const uint4* __restrict__ lay, int64_t KT,
                                                       int kt_cta, const uint4* __restrict__ digits,
                                                       double* __restrict__ out) {
  extern __shared__ uint4 dg[];
  const int ktiles = kt_cta;
  const int64_t kt0 = (int64_t)blockIdx.y * kt_cta;
  for (int i = threadIdx.x; i < ktiles * 64; i += 256) dg[i] = digits[kt0 * 64 + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tid = lane & 3;
  const int64_t strip0 = ((int64_t)blockIdx.x * 8 + warp) * R;
  const uint4* src = lay + (strip0 * KT + kt0) * 32 + lane;
  int acc[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0;
  uint4 buf[DEPTH][R];
#pragma unroll
  for (int d = 0; d < DEPTH; ++d)
#pragma unroll
    for (int r = 0; r < R; ++r) buf[d][r] = __ldcs(src + r * KT * 32 + d * 32);
  const uint32_t m = 0x03030303u;
  for (int kt = 0; kt < ktiles; kt += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const uint4 b01 = dg[((kt + d) * 8 + tid) * 8 + g];
      const uint4 b23 = dg[((kt + d) * 8 + tid + 4) * 8 + g];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint4 w = buf[d][r];
        if (kt + d + DEPTH < ktiles) buf[d][r] = __ldcs(src + r * KT * 32 + (kt + d + DEPTH) * 32);
        mma_u8s8(acc[r], w.x & m, w.y & m, (w.x >> 2) & m, (w.y >> 2) & m, b01.x, b01.y);
        mma_u8s8(acc[r], (w.x >> 4) & m, (w.y >> 4) & m, (w.x >> 6) & m, (w.y >> 6) & m, b01.z, b01.w);
        mma_u8s8(acc[r], w.z & m, w.w & m, (w.z >> 2) & m, (w.w >> 2) & m, b23.x, b23.y);
        mma_u8s8(acc[r], (w.z >> 4) & m, (w.w >> 4) & m, (w.z >> 6) & m, (w.w >> 6) & m, b23.z, b23.w);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    out[((strip0 + r) * gridDim.y + blockIdx.y) * 32 + lane] =
        (double)acc[r][0] + 256.0 * acc[r][1] + (double)acc[r][2] * 3.0 + acc[r][3];
}

int main() {
  int* dout;
  long long* dcyc;
  CK(cudaMalloc(&dout, 148 * 8 * 1024 * sizeof(int)));
  CK(cudaMalloc(&dcyc, 148 * 8 * sizeof(long long)));
  for (int bps : {1, 2, 4, 8}) {
    const int blocks = 148 * bps, threads = 256, iters = 4096;
    mma_rate<8><<<blocks, threads>>>(iters, dout, dcyc);
    CK(cudaDeviceSynchronize());
    std::vector<long long> cyc(blocks);
    CK(cudaMemcpy(cyc.data(), dcyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (auto c : cyc) mx = c > mx ? c : mx;
    const double mmas_per_sm = (double)bps * (threads / 32) * iters * 8;
    printf("mma.sync m16n8k32 u8.s8: %d warps/SM -> %.3f MMA/clk/SM (%.0f int8 MAC/clk/SM)\n",
           bps * 8, mmas_per_sm / mx, mmas_per_sm / mx * 16 * 8 * 32);
  }
  // GEMV prototype: 100k rows x 10k cols (2-bit) = 250 MB
  const int64_t rows = 100000, cols = 10240;
  const int64_t strips = (rows + 15) / 16, KT = cols / 128;
  const int64_t strips_pad = ((strips + 31) / 32) * 32;
  const size_t bytes = (size_t)strips_pad * KT * 512;
  uint4* lay;
  uint4* dig;
  double* out;
  uint4* lay2;
  CK(cudaMalloc(&lay, bytes));
  CK(cudaMemset(lay, 0x55, bytes));
  CK(cudaMalloc(&lay2, bytes));
  CK(cudaMemset(lay2, 0x66, bytes));
  bool alternate = false;
  CK(cudaMalloc(&dig, KT * 64 * 16));
  CK(cudaMemset(dig, 0x11, KT * 64 * 16));
  auto run = [&](auto kern, const char* name, int kt_cta, int rr = 1) -> int {
    const int ny = (int)(KT / kt_cta);
    CK(cudaMalloc(&out, (size_t)strips_pad * ny * 32 * sizeof(double)));
    dim3 grid((unsigned)(strips_pad / 8 / rr), (unsigned)ny);
    const size_t smem = (size_t)kt_cta * 64 * 16;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) kern<<<grid, 256, smem>>>(lay, KT, kt_cta, dig, out);
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
      kern<<<grid, 256, smem>>>((alternate && (r & 1)) ? lay2 : lay, KT, kt_cta, dig, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("gemv proto %s kt_cta=%d: %.4f ms, %.1f GB/s packed\n", name, kt_cta, ms,
           bytes / (ms * 1e6));
    cudaFree(out);
    return 0;
  };
  for (int alt = 0; alt < 2; ++alt) {
    alternate = alt;
    printf("alternate buffers: %d\n", alt);
    run(gemv_proto<4, 4, 0>, "d4 m4 full", 16);
    run(gemv_proto<4, 4, 1>, "d4 m4 noMMA", 16);
    run(gemv_multi<2, 2, 4>, "R2 d2 m4", 16, 2);
    run(gemv_multi<2, 4, 3>, "R2 d4 m3", 16, 2);
  }
  return 0;
}
