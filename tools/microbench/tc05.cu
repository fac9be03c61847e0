// tcgen05 (5th-generation tensor core) u8 x s8 -> s32 check: one CTA,
// D[128 x N] (TMEM) = A[128 x K] (smem, K-major, no swizzle) . B[N x K]^T
// (smem, K-major), compared with the CPU. Validates the instruction and
// shared-memory descriptors the block-product kernel uses.
//   usage: tc05 [N] [K] [variant]   variant 0: LBO = K-adjacent core
//   matrices, SBO = M-adjacent (CUTLASS's canonical K-major INTERLEAVE);
//   1: swapped (must fail).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// canonical K-major, no swizzle: core matrix (8 rows x 16 B) (mi, kc) at
// mi * SBO + kc * LBO; here LBO = 128 (K chunks adjacent), SBO = kchunks * 128
__device__ __forceinline__ uint32_t core_off(int row, int kbyte, int kchunks) {
  return (row >> 3) * (kchunks * 128) + (kbyte >> 4) * 128 + (row & 7) * 16 + (kbyte & 15);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void k_tc05(const uint8_t* A, const int8_t* B, int N, int K, int variant, int* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;                       // 128 x K
  uint8_t* sb = sm + 128 * K;             // N x K
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int kch = K / 16;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    sa[core_off(r, k, kch)] = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    sb[core_off(r, k, kch)] = (uint8_t)B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                     smem_u32(&tbase))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    // instruction descriptor, kind::i8: D s32 (2 << 4), A u8 (0 << 7), B s8 (1 << 10),
    // K-major A and B, N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    const uint32_t lbo = variant == 0 ? 128u : (uint32_t)kch * 128u;
    const uint32_t sbo = variant == 0 ? (uint32_t)kch * 128u : 128u;
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t da = smem_desc(smem_u32(sa) + ks * 256, lbo, sbo);
      const uint64_t db = smem_desc(smem_u32(sb) + ks * 256, lbo, sbo);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W%=;\n}" ::"r"(
          smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // 32x32b.x16: warp w reads TMEM lanes 32w..32w+31, columns 0..15
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(tmem + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const int row = 32 * w + l;
  for (int c = 0; c < 16 && c < N; ++c) D[row * N + c] = (int)r[c];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 16;
  const int K = argc > 2 ? atoi(argv[2]) : 64;
  const int variant = argc > 3 ? atoi(argv[3]) : 0;
  std::vector<uint8_t> A(128 * K);
  std::vector<int8_t> B(N * K);
  for (int i = 0; i < 128 * K; ++i) A[i] = (uint8_t)((i * 37 + 11) % 193);
  for (int i = 0; i < N * K; ++i) B[i] = (int8_t)(((i * 53 + 7) % 255) - 127);
  uint8_t* dA;
  int8_t* dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, sizeof(int) * 128 * N);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, sizeof(int) * 128 * N);
  const int smem = 128 * K + N * K;
  cudaFuncSetAttribute(k_tc05, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_tc05<<<1, 128, smem>>>(dA, dB, N, K, variant, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(e));
    return 2;
  }
  std::vector<int> D(128 * N);
  cudaMemcpy(D.data(), dD, sizeof(int) * D.size(), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N && n < 16; ++n) {
      long long s = 0;
      for (int k = 0; k < K; ++k) s += (long long)A[m * K + k] * (long long)B[n * K + k];
      if (s != D[m * N + n]) {
        if (bad < 5) printf("  mismatch m=%d n=%d: %d vs %lld\n", m, n, D[m * N + n], s);
        ++bad;
      }
    }
  printf("variant %d N=%d K=%d: %s (%d mismatches)\n", variant, N, K, bad ? "FAIL" : "OK", bad);
  return bad ? 1 : 0;
}
