// Streaming experiment for the packed product main loop:
// register streaming (the k_pm_main loop: 8 warps x 2 strips, two tiles of
// register prefetch per strip, 14-tile ranges) against a persistent CTA whose
// producer warp streams whole strip ranges (7 KB or 3.5 KB contiguous) into a
// shared-memory ring with cp.async.bulk on full/empty mbarriers, consumers
// reading the A tiles from shared memory. Config-4 K2 geometry: 500,000 rows
// (31,264 strips) x 784 tiles = 12.55 GB, larger than L2. Digits constant
// (the loop cost is what is measured; no epilogue beyond one store per row).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o ring ring.cu
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

constexpr int kFull = 14;

__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_tile(int (&acc)[4], const uint4 w, const uint4 b01,
                                         const uint4 b23) {
  const uint32_t m0 = 0x03030303u, m1 = m0 << 2, m2 = m0 << 4, m3 = m0 << 6;
  mma_u8s8(acc, w.x & m0, w.y & m0, w.x & m1, w.y & m1, b01.x, b01.y);
  mma_u8s8(acc, w.x & m2, w.y & m2, w.x & m3, w.y & m3, b01.z, b01.w);
  mma_u8s8(acc, w.z & m0, w.w & m0, w.z & m1, w.w & m1, b23.x, b23.y);
  mma_u8s8(acc, w.z & m2, w.w & m2, w.z & m3, w.w & m3, b23.z, b23.w);
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// (a) register streaming: grid (row blocks, nkc), 8 warps x 2 strips, tiles
// t+1, t+2 in flight per strip, fully unrolled 14-tile loop (k_pm_main's loop)
__global__ void __launch_bounds__(256, 4) k_reg(const uint4* __restrict__ lay, int64_t KT,
                                               const uint4* __restrict__ dig,
                                               int* __restrict__ out) {
  __shared__ uint4 dg[kFull * 64];
  const int kc = blockIdx.y, bx = blockIdx.x;
  const int64_t kt0 = (int64_t)kc * kFull;
  for (int i = threadIdx.x; i < kFull * 64; i += 256) dg[i] = dig[kt0 * 64 + i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tid = lane & 3;
  const int64_t strip0 = ((int64_t)bx * 8 + warp) * 2;
  const uint4* p0 = lay + (strip0 * KT + kt0) * 32 + lane;
  const uint4* p1 = p0 + KT * 32;
  int acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  uint4 bA[2], bB[2], bC[2];
  bA[0] = ld_stream(p0);
  bA[1] = ld_stream(p1);
  bB[0] = ld_stream(p0 + 32);
  bB[1] = ld_stream(p1 + 32);
  __syncthreads();
  const int sw = g ^ (2 * tid);
  const uint4* bp = dg + tid * 8 + sw;
#define STEP(T, CUR, DST)                                      \
  {                                                            \
    const uint4 b01 = bp[(T) * 64], b23 = bp[(T) * 64 + 32];   \
    if ((T) + 2 < kFull) {                                     \
      DST[0] = ld_stream(p0 + ((T) + 2) * 32);                 \
      DST[1] = ld_stream(p1 + ((T) + 2) * 32);                 \
    }                                                          \
    mma_tile(acc[0], CUR[0], b01, b23);                        \
    mma_tile(acc[1], CUR[1], b01, b23);                        \
  }
#pragma unroll
  for (int T = 0; T < kFull; T += 3) {
    STEP(T, bA, bC)
    if (T + 1 < kFull) STEP(T + 1, bB, bA)
    if (T + 2 < kFull) STEP(T + 2, bC, bB)
  }
#undef STEP
  const int64_t b = (int64_t)kc * gridDim.x + bx;
  out[(b * 8 + warp) * 32 + lane] = acc[0][0] + acc[0][1] * 3 + acc[0][2] * 5 + acc[0][3] * 7 +
                                    acc[1][0] + acc[1][1] * 11 + acc[1][2] * 13 + acc[1][3];
}

// (b) persistent ring. CTA = 8 consumer warps + 1 producer warp; work units
// (row block bx, range kc) in kc-major order, CTA c takes a contiguous chunk.
// Stage = SPS tiles of a warp's two strips (2 bulk copies of SPS * 512 B);
// each consumer warp has its own ring of R stages (a slot's previous use was
// the same warp's, so a parity wait can never alias an older phase).
template <int SPS, int R>
__global__ void __launch_bounds__(288, 1) k_ring(const uint4* __restrict__ lay, int64_t KT,
                                                int nbx, int64_t units,
                                                const uint4* __restrict__ dig,
                                                int* __restrict__ out) {
  constexpr int kStrip = SPS * 512;
  constexpr int kHalves = kFull / SPS;  // stages per warp per unit
  constexpr int NS = 8 * R;
  extern __shared__ __align__(128) uint4 smem[];
  uint4* ring = smem;                      // NS * 2 * SPS * 32 uint4
  uint4* dg = smem + NS * 2 * SPS * 32;    // kFull * 64 uint4 (constant digits)
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < kFull * 64; i += blockDim.x) dg[i] = dig[i];
  __syncthreads();
  if (warp == 8) {  // producer
    if (lane == 0) {
      int64_t j = 0;  // per-warp stage sequence number
      for (int64_t u = u0; u < u1; ++u) {
        const int64_t kc = u / nbx, bx = u - kc * nbx;
        for (int h = 0; h < kHalves; ++h, ++j)
          for (int w = 0; w < 8; ++w) {
            const int slot = w * R + (int)(j % R);
            if (j >= R) mbar_wait(&empty[slot], (uint32_t)(((j / R) & 1) ^ 1));
            const int64_t strip = bx * 16 + 2 * w;
            const uint4* src = lay + (strip * KT + kc * kFull + h * SPS) * 32;
            uint4* dst = ring + slot * 2 * SPS * 32;
            mbar_arrive_expect_tx(&full[slot], 2 * kStrip);
            bulk_g2s(dst, src, kStrip, &full[slot]);
            bulk_g2s(dst + SPS * 32, src + KT * 32, kStrip, &full[slot]);
          }
      }
    }
    return;
  }
  const int g = lane >> 2, tid = lane & 3;
  const int sw = g ^ (2 * tid);
  int64_t j = 0;
  for (int64_t u = u0; u < u1; ++u) {
    int acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    const uint4* bp = dg + tid * 8 + sw;
#pragma unroll
    for (int h = 0; h < kHalves; ++h, ++j) {
      const int slot = warp * R + (int)(j % R);
      mbar_wait(&full[slot], (uint32_t)((j / R) & 1));
      const uint4* a0 = ring + slot * 2 * SPS * 32 + lane;
      const uint4* a1 = a0 + SPS * 32;
#pragma unroll
      for (int t = 0; t < SPS; ++t) {
        const uint4 b01 = bp[(h * SPS + t) * 64], b23 = bp[(h * SPS + t) * 64 + 32];
        const uint4 w0 = a0[t * 32], w1 = a1[t * 32];
        mma_tile(acc[0], w0, b01, b23);
        mma_tile(acc[1], w1, b01, b23);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    out[(u * 8 + warp) * 32 + lane] = acc[0][0] + acc[0][1] * 3 + acc[0][2] * 5 +
                                      acc[0][3] * 7 + acc[1][0] + acc[1][1] * 11 +
                                      acc[1][2] * 13 + acc[1][3];
  }
}

// (c) self-fed rings: no producer warp; each warp's lane 0 issues the bulk
// copies of its own stages and refills a slot right after consuming it
// (8 issuing threads per SM, no empty barriers).
template <int SPS, int R>
__global__ void __launch_bounds__(256, 1) k_self(const uint4* __restrict__ lay, int64_t KT,
                                                int nbx, int64_t units,
                                                const uint4* __restrict__ dig,
                                                int* __restrict__ out) {
  constexpr int kStrip = SPS * 512;
  constexpr int kHalves = kFull / SPS;
  constexpr int NS = 8 * R;
  extern __shared__ __align__(128) uint4 smem[];
  uint4* ring = smem;
  uint4* dg = smem + NS * 2 * SPS * 32;
  __shared__ __align__(8) uint64_t full[NS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
  const int64_t jend = (u1 - u0) * kHalves;
  if (lane == 0)
    for (int s = 0; s < R; ++s) mbar_init(&full[warp * R + s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int64_t j) {  // lane 0: stage j of this warp
    const int64_t u = u0 + j / kHalves;
    const int h = (int)(j % kHalves);
    const int64_t kc = u / nbx, bx = u - kc * nbx;
    const int64_t strip = bx * 16 + 2 * warp;
    const uint4* src = lay + (strip * KT + kc * kFull + h * SPS) * 32;
    const int slot = warp * R + (int)(j % R);
    uint4* dst = ring + slot * 2 * SPS * 32;
    mbar_arrive_expect_tx(&full[slot], 2 * kStrip);
    bulk_g2s(dst, src, kStrip, &full[slot]);
    bulk_g2s(dst + SPS * 32, src + KT * 32, kStrip, &full[slot]);
  };
  if (lane == 0)
    for (int64_t j = 0; j < R && j < jend; ++j) issue(j);
  for (int i = threadIdx.x; i < kFull * 64; i += blockDim.x) dg[i] = dig[i];
  __syncthreads();
  const int g = lane >> 2, tid = lane & 3;
  const int sw = g ^ (2 * tid);
  int64_t j = 0;
  for (int64_t u = u0; u < u1; ++u) {
    int acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    const uint4* bp = dg + tid * 8 + sw;
#pragma unroll
    for (int h = 0; h < kHalves; ++h, ++j) {
      const int slot = warp * R + (int)(j % R);
      mbar_wait(&full[slot], (uint32_t)((j / R) & 1));
      const uint4* a0 = ring + slot * 2 * SPS * 32 + lane;
      const uint4* a1 = a0 + SPS * 32;
#pragma unroll
      for (int t = 0; t < SPS; ++t) {
        const uint4 b01 = bp[(h * SPS + t) * 64], b23 = bp[(h * SPS + t) * 64 + 32];
        const uint4 w0 = a0[t * 32], w1 = a1[t * 32];
        mma_tile(acc[0], w0, b01, b23);
        mma_tile(acc[1], w1, b01, b23);
      }
      __syncwarp();
      if (lane == 0 && j + R < jend) issue(j + R);
    }
    out[(u * 8 + warp) * 32 + lane] = acc[0][0] + acc[0][1] * 3 + acc[0][2] * 5 +
                                      acc[0][3] * 7 + acc[1][0] + acc[1][1] * 11 +
                                      acc[1][2] * 13 + acc[1][3];
  }
}

__global__ void k_fill(uint32_t* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29;
    x *= 0xBF58476D1CE4E5B9ull;
    p[i] = (uint32_t)(x >> 32);
  }
}

// plain streaming read (the copy-peak reference for a read-only stream)
__global__ void k_read(const uint4* __restrict__ p, int64_t n, uint32_t* out) {
  uint32_t x = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = ld_stream(p + i);
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x12345678u) out[0] = x;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 40;
  const int64_t ulim = argc > 2 ? atoll(argv[2]) : 0;
  const int64_t strips = 31264, KT = 784, nbx = strips / 16, nkc = KT / kFull;
  const size_t bytes = (size_t)strips * KT * 512;
  uint4 *lay, *dig;
  int* out;
  uint32_t* dummy;
  CK(cudaMalloc(&lay, bytes));
  CK(cudaMemset(lay, 0x5a, bytes));
  CK(cudaMalloc(&dig, KT * 64 * 16));
  CK(cudaMemset(dig, 0x11, KT * 64 * 16));
  CK(cudaMalloc(&out, (size_t)nbx * nkc * 8 * 32 * sizeof(int)));
  CK(cudaMalloc(&dummy, 16));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch, const char* name) -> int {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-28s %.4f ms  %.1f GB/s\n", name, ms, bytes / (ms * 1e6));
    return 0;
  };
  const int64_t units = ulim ? ulim : nbx * nkc;
  // correctness: the ring kernels' per-row sums against the register kernel's
  std::vector<int> ref((size_t)nbx * nkc * 256), got((size_t)nbx * nkc * 256);
  k_fill<<<148 * 8, 256>>>(reinterpret_cast<uint32_t*>(lay), (int64_t)(bytes / 4));
  CK(cudaDeviceSynchronize());
  k_reg<<<dim3(nbx, nkc), 256>>>(lay, KT, dig, out);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(ref.data(), out, ref.size() * sizeof(int), cudaMemcpyDeviceToHost));
  auto check = [&](auto launch, const char* name) -> int {
    CK(cudaMemset(out, 0, got.size() * sizeof(int)));
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(got.data(), out, got.size() * sizeof(int), cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t i = 0; i < units * 256; ++i) bad += got[i] != ref[i];
    printf("%-28s check: %lld mismatches of %lld\n", name, (long long)bad, (long long)(units * 256));
    return 0;
  };
  auto ring7 = k_ring<7, 3>;    // 7 KB stages, 3 per warp (168 KB)
  auto ring2 = k_ring<2, 10>;   // 2 KB stages, 10 per warp (160 KB)
  auto ring1 = k_ring<1, 20>;   // 1 KB stages, 20 per warp (160 KB)
  const size_t sm7 = (size_t)24 * 7 * 1024 + kFull * 1024;
  const size_t sm2 = (size_t)80 * 2 * 1024 + kFull * 1024;
  const size_t sm1 = (size_t)160 * 1 * 1024 + kFull * 1024;
  CK(cudaFuncSetAttribute(ring7, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm7));
  CK(cudaFuncSetAttribute(ring2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
  auto self7 = k_self<7, 3>;
  auto self2 = k_self<2, 10>;
  CK(cudaFuncSetAttribute(self7, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm7));
  CK(cudaFuncSetAttribute(self2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
  CK(cudaFuncSetAttribute(ring1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
  printf("layout %.2f GB, %lld units\n", bytes / 1e9, (long long)units);
  check([&] { ring7<<<148, 288, sm7>>>(lay, KT, nbx, units, dig, out); }, "ring 7KB x3");
  check([&] { ring2<<<148, 288, sm2>>>(lay, KT, nbx, units, dig, out); }, "ring 2KB x10");
  check([&] { self7<<<148, 256, sm7>>>(lay, KT, nbx, units, dig, out); }, "self 7KB x3");
  check([&] { self2<<<148, 256, sm2>>>(lay, KT, nbx, units, dig, out); }, "self 2KB x10");
  check([&] { ring1<<<148, 288, sm1>>>(lay, KT, nbx, units, dig, out); }, "ring 1KB x20");
  for (int pass = 0; pass < 2; ++pass) {
    timeit([&] { k_read<<<148 * 8, 512>>>(lay, (int64_t)(bytes / 16), dummy); }, "read");
    timeit([&] { k_reg<<<dim3(nbx, nkc), 256>>>(lay, KT, dig, out); }, "register stream");
    timeit([&] { ring7<<<148, 288, sm7>>>(lay, KT, nbx, units, dig, out); }, "ring 7KB x3");
    timeit([&] { ring2<<<148, 288, sm2>>>(lay, KT, nbx, units, dig, out); }, "ring 2KB x10");
    timeit([&] { self7<<<148, 256, sm7>>>(lay, KT, nbx, units, dig, out); }, "self 7KB x3");
    timeit([&] { self2<<<148, 256, sm2>>>(lay, KT, nbx, units, dig, out); }, "self 2KB x10");
    timeit([&] { ring1<<<148, 288, sm1>>>(lay, KT, nbx, units, dig, out); }, "ring 1KB x20");
  }
  return 0;
}
