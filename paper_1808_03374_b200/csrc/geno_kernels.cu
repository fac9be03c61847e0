// Packed-genotype kernels for sm_100a: tile-layout build (K8), marker counts
// (K7), per-CTA missing lists, coefficient digitization, and the packed
// matrix-vector products
//   K1 = reference apply         (X x,   per-SNP dot:   rows = SNPs,    cols = samples)
//   K2 = reference apply_adjoint (X^T y, per-sample sum: rows = samples, cols = SNPs)
// which are one kernel (k_pm_main) over two tile layouts of the same matrix.
//
// Reference semantics (/root/reference/proj):
//   .bed code table            genio.cpp:33   (00->2, 01->missing, 10->1, 11->0)
//   standardized entry          genio.cpp:124-185: (d - mu_j)/s_j, missing -> 0
//   DenseOperator apply/adjoint linop.hpp:50-58
//
// Arithmetic: exact fixed-point digits on the tensor
// cores. For one CTA's column range (kt_cta tiles of 128 columns; 14 tiles =
// 1792 columns by default) the fp64 coefficients v_c are rounded to 62-bit
// fixed point relative to the range's largest exponent E, M_c = rn(v_c 2^(62-E)),
// and split into 8 balanced base-256 digits d_i(c) in [-128, 127]. The 2-bit dosage codes a_rc in {0,1,2,3} (3 =
// missing) are expanded to u8 fragment registers and
//   D_i(r) = sum_c a_rc d_i(c)
// is accumulated EXACTLY in int32 by mma.sync.m16n8k32 (u8 x s8 -> s32; the
// MMA's N = 8 is the 8 digits). The row value is 2^(E-62) sum_i D_i 256^i,
// formed in fp64 (one rounding per partial; the only other error is the
// 2^-63-relative rounding of the coefficients), which is at least as accurate
// as the reference's fp64 dot products. Integer sums are order-free, and the
// few fp64 combinations are in a fixed order, so results are bitwise
// reproducible run to run.
//
// Missing entries stay r = 3 in the layouts (the layouts keep the full .bed
// information); their contribution is removed exactly in the main kernel's
// epilogue from the CTA's own sorted missing list (16-bit local column
// indices), together with the mean term:
//   K1: y_j = inv_s_j (sum_s a_js x_s - mu_j X - (3 - m_j) sum_{s miss} x_s)
//   K2: z_s = sum_j c_j a_js - sum_j c_j mu_j - sum_{j miss} c_j (3 - m_j),  c_j = inv_s_j y_j
// m_j = observed mean = the value impute_mean gives a missing entry
// (genio.cpp:144); m_j = mu_j for the standardizing schemes, so missing
// entries are 0 there, and the raw mean-imputed value for scheme none.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"
#include "pdl.hpp"

namespace gkb {
namespace dev {

namespace {

constexpr int kThreads = 256;
#ifndef GKB_SPW
#define GKB_SPW 2
#endif
constexpr int kStripsPerWarp = GKB_SPW;  // row strips sharing each B fragment
constexpr int kDepth = 2;                // tiles in flight per strip
#ifndef GKB_FULL
#define GKB_FULL 14
#endif
constexpr int kFullRange = GKB_FULL;  // pm_plan's default kt_cta: fully unrolled main loop
static_assert(kStripsPerWarp <= 2, "the unrolled full-range loop prefetches strips 0 and 1");
constexpr int kRowsPerCta = 8 * kStripsPerWarp * 16;  // 256
constexpr int kStripsPerCta = 8 * kStripsPerWarp;
constexpr int kMinCtas = kStripsPerWarp <= 2 ? 4 : 3;  // per SM (register budget)
#ifndef GKB_BULK_STAGE
#define GKB_BULK_STAGE 1  // k_pm_main: bulk-copy (TMA engine) staging on an mbarrier
#endif
#ifndef GKB_EARLY_STAGE
#define GKB_EARLY_STAGE 1  // k_pm_main: staging complete before the loop (no barrier after it)
#endif

// .bed 2-bit code -> dosage code r (r_hi = ~h, r_lo = l ^ h per field).
__device__ __forceinline__ uint32_t bed_to_r(uint32_t c) {
  return ((~c) & 0xAAAAAAAAu) | ((c ^ (c >> 1)) & 0x55555555u);
}
// inverse mapping r -> .bed code
__device__ __forceinline__ uint32_t r_to_bed(uint32_t r) {
  return ((~r) & 0xAAAAAAAAu) | ((r ^ ((~r) >> 1)) & 0x55555555u);
}
__device__ __forceinline__ uint32_t missing_mask(uint32_t r) { return r & (r >> 1) & 0x55555555u; }

// Programmatic dependent launch (pdl.hpp). The product kernels (digitize ->
// main -> reduce) run only work on data that is immutable for the whole solve
// (tile layouts, missing lists) before pdl_wait().

#ifndef GKB_L2PF
#define GKB_L2PF 0
#endif
constexpr int kL2Pf = GKB_L2PF;  // L2 prefetch distance in tiles (0: off)
// one 512-byte tile into L2 (bulk prefetch, no registers, no completion)
__device__ __forceinline__ void prefetch_l2_512(const uint4* p) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;" ::"l"(p) : "memory");
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// 32-bit word (row, word-column wc) of a tile layout: strips of 16 rows,
// K tiles of 8 words (128 columns); tile = 512 B in mma fragment order,
// uint4 #(4g + t) = {(g, t), (g+8, t), (g, t+4), (g+8, t+4)} (row, word in tile).
__device__ __forceinline__ int64_t word_index(int64_t KT, int64_t row, int64_t wc) {
  const int64_t s = row >> 4;
  const int gg = (int)(row & 15), g = gg & 7, half = gg >> 3;
  const int64_t kt = wc >> 3;
  const int q = (int)(wc & 7), t = q & 3, hi = q >> 2;
  return ((s * KT + kt) * 32 + 4 * g + t) * 4 + half + 2 * hi;
}

// Deterministic block sum (fixed shuffle tree, then warps in order).
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    red[32] = t;
  }
  __syncthreads();
  return red[32];
}

__device__ int block_max_int(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_down_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) t = max(t, red[i]);
    red[32] = t;
  }
  __syncthreads();
  return red[32];
}

__device__ __forceinline__ int exp_of(double v) {
  if (v == 0.0) return -1100;
  int e;
  frexp(v, &e);
  return e;
}

__device__ __forceinline__ double pow2(int k) {  // exact 2^k, -1022 <= k <= 1023
  return __hiloint2double((1023 + k) << 20, 0);
}

// scalbn(v, k) with one DMUL when 2^k is a normal double (then v * 2^k is the
// exact product rounded once, like scalbn); the library call otherwise
__device__ __forceinline__ double scale2(double v, int k) {
  return (k >= -1022 && k <= 1023) ? v * pow2(k) : scalbn(v, k);
}

// ---------------------------------------------------------------- K8 / K7
// .bed records of one staging block (rows [row0, row0+rows) of the shard)
// -> layout 1 (rows = SNPs): thread per (SNP row, word of 16 samples).
__global__ void k_build_lt1(const uint8_t* __restrict__ bed, int64_t stride, int64_t rows,
                            int64_t row0, int64_t n, int64_t W, int64_t KT,
                            uint32_t* __restrict__ lay) {
  const int64_t total = rows * W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = idx / W, w = idx - rr * W;
    const int64_t valid = n - 16 * w;
    const uint32_t pad_mask = valid >= 16 ? 0xFFFFFFFFu : ((1u << (2 * valid)) - 1u);
    const uint8_t* rec = bed + rr * stride;
    uint32_t v = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * w + t < stride) v |= (uint32_t)rec[4 * w + t] << (8 * t);
    lay[word_index(KT, row0 + rr, w)] = bed_to_r(v) & pad_mask;
  }
}

// -> layout 2 (rows = samples, cols = SNPs): thread per (group of 16 SNP rows,
// word of 16 samples); a 16 x 16 transpose of 2-bit fields. row0 % 16 == 0.
__global__ void k_build_lt2(const uint8_t* __restrict__ bed, int64_t stride, int64_t rows,
                            int64_t row0, int64_t n, int64_t W, int64_t KT,
                            uint32_t* __restrict__ lay) {
  const int64_t groups = (rows + 15) / 16;
  const int64_t total = groups * W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jg = idx / W, w = idx - jg * W;
    const int64_t valid = n - 16 * w;
    const uint32_t pad_mask = valid >= 16 ? 0xFFFFFFFFu : ((1u << (2 * valid)) - 1u);
    uint32_t out[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) out[k] = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t rr = 16 * jg + i;
      uint32_t v = 0;
      if (rr < rows) {
        const uint8_t* rec = bed + rr * stride;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * w + t < stride) v |= (uint32_t)rec[4 * w + t] << (8 * t);
        v = bed_to_r(v) & pad_mask;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) out[k] |= ((v >> (2 * k)) & 3u) << (2 * i);
    }
    const int64_t wc = (row0 >> 4) + jg;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t s = 16 * w + k;
      if (s < n) lay[word_index(KT, s, wc)] = out[k];
    }
  }
}

// one warp per SNP row of layout 1: [n0, n1, n2, nmiss]
__global__ void k_marker_counts(const uint32_t* __restrict__ lay, int64_t KT, int64_t p_loc,
                                int64_t W, int64_t n, int64_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < p_loc; j += warps) {
    int c1 = 0, c2 = 0, c3 = 0;
    for (int64_t w = lane; w < W; w += 32) {
      const uint32_t r = lay[word_index(KT, j, w)], hi = (r >> 1) & 0x55555555u,
                     lo = r & 0x55555555u;
      c3 += __popc(hi & lo);
      c2 += __popc(hi & ~lo);
      c1 += __popc(~hi & lo & 0x55555555u);
    }
    for (int o = 16; o > 0; o >>= 1) {
      c1 += __shfl_down_sync(0xffffffffu, c1, o);
      c2 += __shfl_down_sync(0xffffffffu, c2, o);
      c3 += __shfl_down_sync(0xffffffffu, c3, o);
    }
    if (lane == 0) {
      counts[4 * j + 0] = n - c1 - c2 - c3;
      counts[4 * j + 1] = c1;
      counts[4 * j + 2] = c2;
      counts[4 * j + 3] = c3;
    }
  }
}

__global__ void k_layout_to_bed(const uint32_t* __restrict__ lay, int64_t KT, int64_t n,
                                int64_t row0, int64_t nrows, uint8_t* __restrict__ out) {
  const int64_t stride = (n + 3) / 4, W = (n + 15) / 16;
  const int64_t total = nrows * W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = idx / W, w = idx - rr * W;
    uint32_t c = r_to_bed(lay[word_index(KT, row0 + rr, w)]);
    const int64_t valid = n - 16 * w;
    if (valid < 16) c &= (1u << (2 * valid)) - 1u;  // pads 00 (genio.cpp:100)
    uint8_t* rec = out + rr * stride;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * w + t < stride) rec[4 * w + t] = (uint8_t)(c >> (8 * t));
  }
}

// ---------------------------------------------------------------- missing lists
// Per-CTA missing lists: block b = kc * grid_x + bx
// covers rows [256 bx, 256 bx + 256) x columns [128 kt_cta kc, 128 kt_cta (kc + 1)) of a
// tile layout -- exactly one k_pm_main CTA. Row r of the block owns
//   ent[base[b] + off[b*257 + r] .. base[b] + off[b*257 + r + 1])
// = the block-local column indices (< 128 kt_cta = 1792 by default, ascending) of its missing entries.
// Count pass (kFill = false) writes cnt[b*256 + r]; fill pass writes ent.
template <bool kFill>
__global__ void __launch_bounds__(kRowsPerCta) k_miss_tiles(const uint32_t* __restrict__ lay, int64_t KT,
                                                    int kt_cta, uint32_t* __restrict__ cnt,
                                                    const uint32_t* __restrict__ off,
                                                    const int64_t* __restrict__ base,
                                                    uint16_t* __restrict__ ent) {
  const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int r = threadIdx.x;
  const int64_t row = (int64_t)blockIdx.x * kRowsPerCta + r;
  const int64_t wc0 = (int64_t)blockIdx.y * kt_cta * 8;
  const int64_t wc1 = min(KT * 8, wc0 + (int64_t)kt_cta * 8);
  uint32_t c = 0;
  int64_t pos = kFill ? base[b] + off[b * (kRowsPerCta + 1) + r] : 0;
  for (int64_t wc = wc0; wc < wc1; ++wc) {
    uint32_t m = missing_mask(lay[word_index(KT, row, wc)]);
    if (kFill) {
      while (m) {
        const int bit = __ffs(m) - 1;
        ent[pos++] = (uint16_t)(16 * (wc - wc0) + (bit >> 1));
        m &= m - 1;
      }
    } else {
      c += __popc(m);
    }
  }
  if (!kFill) cnt[b * kRowsPerCta + r] = c;
}

// CTA per block: exclusive scan of the block's span counts -> off, block total -> tot.
__global__ void __launch_bounds__(512) k_block_scan(const uint32_t* __restrict__ cnt, int span,
                                                    uint32_t* __restrict__ off,
                                                    int64_t* __restrict__ tot) {
  __shared__ uint32_t s[512];
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  s[t] = t < span ? cnt[b * span + t] : 0u;
  __syncthreads();
  for (int o = 1; o < 512; o <<= 1) {
    const uint32_t v = t >= o ? s[t - o] : 0u;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  if (t == 0) off[b * (span + 1)] = 0;
  if (t < span) off[b * (span + 1) + t + 1] = s[t];
  if (t == span - 1) tot[b] = s[t];
}

// ---------------------------------------------------------------- digitize
// One CTA per column range kc (kt_cta * 128 columns): coefficients v_c
//   MODE 0 (K1): v_c = x_c,            sum = sum_c v_c           (X of the range)
//   MODE 1 (K2): v_c = inv_s_c * y_c,  sum = sum_c v_c mu_c, cm_c = v_c (3 - mean_c)
//   MODE 2 (K2 from layout 1, single-layout mode): as MODE 1, digits in the
//          k_pm_adj_l1 fragment order
// -> E (largest exponent), 8 balanced base-256 digits of rn(v 2^(62-E)) in
// mma B-fragment order: uint4 (word-column wc, digit i) holds, in 32-bit word
// q, byte e = digit i of column 16 wc + 4 e + q.
template <int MODE>
__global__ void __launch_bounds__(1024) k_digitize(const double* __restrict__ v_in,
                                                   const double* __restrict__ inv_s,
                                                   const double* __restrict__ mu,
                                                   const double* __restrict__ mean, int64_t C,
                                                   int kt_cta, uint4* __restrict__ dig,
                                                   int* __restrict__ dexp,
                                                   double* __restrict__ dsum,
                                                   double* __restrict__ cm,
                                                   const double* __restrict__ div,
                                                   double* __restrict__ store,
                                                   const int* __restrict__ gate,
                                                   uint4* __restrict__ dig2 = nullptr,
                                                   int* __restrict__ dexp2 = nullptr) {
  // kt_cta * 64 uint4 (digits), then kt_cta * 128 doubles; with dig2 (MODE 1,
  // dense-missing mode: the digits of cm as k_digitize<0> would make them from
  // the stored cm, in the same launch) another kt_cta * 64 uint4 + kt_cta * 128 doubles
  extern __shared__ uint4 dsm[];
  __shared__ double red[33];
  __shared__ int redi[33];
  double* vals = reinterpret_cast<double*>(dsm + kt_cta * 64);
  uint8_t* db = reinterpret_cast<uint8_t*>(dsm);
  const bool two = MODE == 1 && dig2 != nullptr;
  uint4* dsm2 = dsm + kt_cta * 64 + kt_cta * 64;  // after vals (kt_cta * 128 doubles)
  double* cvals = reinterpret_cast<double*>(dsm2 + kt_cta * 64);
  int emax2 = -1100;
  // trigger only after the wait: the main kernel's early reads of the lists and
  // layout then follow the completion of every kernel before this one
  pdl_wait();
  pdl_trigger();
  const int kc = blockIdx.x;
  const int ncol = kt_cta * 128;
  const int64_t c0 = (int64_t)kc * ncol;
  int emax = -1100;
  double part = 0.0;
  // div: the input is v_in / *div (the Lanczos normalization w / alpha, z / beta,
  // as k_div_copy_dev divides), stored to `store` unless *gate == 0
  const double dv = div ? *div : 1.0;
  const bool st = div && store && !(gate && *gate == 0);
  for (int t = threadIdx.x; t < ncol; t += blockDim.x) {
    const int64_t c = c0 + t;
    double v = 0.0;
    if (c < C) {
      double x = v_in[c];
      if (div) {
        x = x / dv;
        if (st) store[c] = x;
      }
      if (MODE == 0) {
        v = x;
        part += v;
      } else {  // MODE 1 and 2: the adjoint's coefficients
        v = inv_s[c] * x;
        part += v * mu[c];
        const double cmc = v * (3.0 - mean[c]);  // a missing entry holds the imputed mean (genio.cpp:144)
        cm[c] = cmc;
        if (two) {
          cvals[t] = cmc;
          emax2 = max(emax2, exp_of(cmc));
        }
      }
    } else if (two) {
      cvals[t] = 0.0;
    }
    emax = max(emax, exp_of(v));
    vals[t] = v;
  }
  const int E = block_max_int(emax, redi);
  const double s = block_sum(part, red);
  const int E2 = two ? block_max_int(emax2, redi) : 0;
  if (two) {  // k_digitize<0>'s digits of cm (group-q prescale, swizzled slots)
    uint8_t* db2 = reinterpret_cast<uint8_t*>(dsm2);
    for (int t = threadIdx.x; t < ncol; t += blockDim.x) {
      const int wc = t >> 4, k = t & 15, q = k & 3, e = k >> 2;
      long long M = __double2ll_rn(scale2(cvals[t], 62 - E2 - 2 * q));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int d = (int)(signed char)(M & 0xFF);
        M = (M - d) >> 8;
        db2[(wc * 8 + (i ^ (2 * (wc & 3)))) * 16 + 4 * q + e] = (uint8_t)d;
      }
    }
  }
  for (int t = threadIdx.x; t < ncol; t += blockDim.x) {
    if (MODE == 2) {
      // K2 from layout 1 (k_pm_adj_l1): no column prescale (the 4^q scale sits
      // on the output rows); SNP r of a 16-SNP strip is k-group (r & 7) >> 1,
      // position (r & 1) + 2 (r >> 3); 128 bytes per strip = [digit][group][pos]
      const int sg = t >> 4, r = t & 15, grp = (r & 7) >> 1, pos = (r & 1) + 2 * (r >> 3);
      long long M = __double2ll_rn(scale2(vals[t], 62 - E));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int d = (int)(signed char)(M & 0xFF);
        M = (M - d) >> 8;
        db[sg * 128 + i * 16 + grp * 4 + pos] = (uint8_t)d;
      }
      continue;
    }
    const int wc = t >> 4, k = t & 15, q = k & 3, e = k >> 2;
    // group-q columns meet codes pre-multiplied by 4^q in the MMA (mma_tile)
    long long M = __double2ll_rn(scale2(vals[t], 62 - E - 2 * q));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int d = (int)(signed char)(M & 0xFF);
      M = (M - d) >> 8;
      db[(wc * 8 + (i ^ (2 * (wc & 3)))) * 16 + 4 * q + e] = (uint8_t)d;  // swizzled slot
    }
  }
  __syncthreads();
  uint4* out = dig + (int64_t)kc * kt_cta * 64;
  for (int t = threadIdx.x; t < kt_cta * 64; t += blockDim.x) out[t] = dsm[t];
  if (two) {
    uint4* out2 = dig2 + (int64_t)kc * kt_cta * 64;
    for (int t = threadIdx.x; t < kt_cta * 64; t += blockDim.x) out2[t] = dsm2[t];
  }
  if (threadIdx.x == 0) {
    dexp[kc] = E;
    dsum[kc] = s;
    if (two) dexp2[kc] = E2;
  }
}

// ---------------------------------------------------------------- main
__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// One 512-byte tile (16 rows x 128 columns) against the tile's B fragments:
// each 32-bit word gives four u8 registers w & (0x03030303 << 2q) = 4^q x the
// codes of columns 4e + q of the word (e = byte) -- one LOP3 each, no shifts.
// The 4^q is undone in the digits: k_digitize encodes a group-q column as
// rn(v 2^(62-E-2q)), so every product is code x v x 2^(62-E), exactly.
__device__ __forceinline__ void mma_tile(int (&acc)[4], const uint4 w, const uint4 b01,
                                         const uint4 b23) {
  const uint32_t m0 = 0x03030303u, m1 = m0 << 2, m2 = m0 << 4, m3 = m0 << 6;
  mma_u8s8(acc, w.x & m0, w.y & m0, w.x & m1, w.y & m1, b01.x, b01.y);
  mma_u8s8(acc, w.x & m2, w.y & m2, w.x & m3, w.y & m3, b01.z, b01.w);
  mma_u8s8(acc, w.z & m0, w.w & m0, w.z & m1, w.w & m1, b23.x, b23.y);
  mma_u8s8(acc, w.z & m2, w.w & m2, w.z & m3, w.w & m3, b23.z, b23.w);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }

// Bulk copies on the TMA engine (cp.async.bulk, SASS UBLKCP) completing on an
// mbarrier: one thread stages a CTA's contiguous inputs (digits, correction
// coefficients, missing-list run and offsets) with a handful of instructions
// instead of every thread looping over 4-16 byte copies.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "GKB_MBAR_WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra GKB_MBAR_WAIT%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// dst, src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// sum_{k in [k0, ke)} cv[ent[k]] in order, in one loop of chunks of four with the chunk's loads and adds
// predicated on the run's end (each entry still added in order: same bits),
// so a warp's lanes do not diverge between a chunk loop and a tail loop
__device__ __forceinline__ double walk_list_u(const uint16_t* __restrict__ ent, uint32_t k0,
                                              uint32_t ke, const double* __restrict__ cv) {
  double corr = 0.0;
  const uint32_t n = ke - k0;
#pragma unroll 1
  for (uint32_t i = 0; i < n; i += 4) {
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u < n) x[u] = cv[ent[k0 + i + u]];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u < n) corr += x[u];
  }
  return corr;
}

// two runs (a warp's two strips) in ONE loop of chunks of four: past a run's
// end a lane reads the zero slot cv[-1] = +0.0 instead. A sum that starts at
// +0.0 never becomes -0.0, so adding +0.0 leaves it unchanged and each run's
// sum is the in-order sum -- without the remainder and tail loops, between
// which a warp's lanes diverged (the epilogue's largest instruction cost).
__device__ __forceinline__ void walk_list_pair_u(const uint16_t* __restrict__ ent, uint32_t ka,
                                                 uint32_t kea, uint32_t kb, uint32_t keb,
                                                 const double* __restrict__ cv, double& ca,
                                                 double& cb) {
  double sa = 0.0, sb = 0.0;
  const uint32_t na = kea - ka, nb = keb - kb, n = max(na, nb);
#pragma unroll 1
  for (uint32_t i = 0; i < n; i += 4) {
    int a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = i + u < na ? (int)ent[ka + i + u] : -1;
      b[u] = i + u < nb ? (int)ent[kb + i + u] : -1;
    }
    double x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = cv[a[u]];
      y[u] = cv[b[u]];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      sa += x[u];
      sb += y[u];
    }
  }
  ca = sa;
  cb = sb;
}

// Missing-list staging in shared memory (after the digits): 257 offsets and
// up to kEntCap entries of the CTA's list (longer lists are read from global).
constexpr int kEntCap = 4096 * kStripsPerWarp;
constexpr int kOffBytes = ((kRowsPerCta + 1) * 4 + 15) / 16 * 16;
size_t pm_smem_bytes(int kt_cta) {
  return (size_t)kt_cta * 64 * 16 + kOffBytes + 2 * kEntCap + 16 + (size_t)kt_cta * 128 * 8;
}

// grid (S / 16, nkc). CTA = 8 warps x 2 strips (256 rows) x one column range
// of kt_cta tiles; B fragments (digits) of the range in shared memory, shared
// by the 8 warps and reused across each warp's 2 strips. Writes the range's
// exact partial (MODE 0: K1, MODE 1: K2 -- see the header) to part[kc][row].
// The CTA's missing list (offsets + entries) and the range's correction
// coefficients cval (K1: x, K2: c_j (3 - mu_j)) are staged into shared memory
// by bulk copies in the prologue (below), so the epilogue walk never touches global
// memory (random 8-byte gathers from L2 cost ~30% of the kernel otherwise).
template <int MODE>
__global__ void __launch_bounds__(kThreads, kMinCtas) k_pm_main(
    const uint4* __restrict__ lay, int64_t KT, int kt_cta, const uint4* __restrict__ dig,
    const int* __restrict__ dexp, const double* __restrict__ dsum,
    const double* __restrict__ cval, const double* __restrict__ mu,
    const double* __restrict__ mean, const uint32_t* __restrict__ m_off,
    const int64_t* __restrict__ m_base, const uint16_t* __restrict__ m_ent, int64_t rows_pad,
    int64_t C, double* __restrict__ part, unsigned* __restrict__ tick,
    const double* __restrict__ inv_s, double* __restrict__ yout, int64_t R) {
  extern __shared__ __align__(16) uint4 dg[];  // kt_cta * 64 digits, then list staging
  // grid: (nkc, row blocks) when the reduce is fused (tick != null: the ranges
  // of one row block are adjacent in launch order), else (row blocks, nkc)
  const int kc = tick ? blockIdx.x : blockIdx.y;
  const int bx = tick ? blockIdx.y : blockIdx.x;
  const int nbx = tick ? gridDim.y : gridDim.x;
  const int nkc = tick ? gridDim.x : gridDim.y;
  const int64_t kt0 = (int64_t)kc * kt_cta;
  const int ktiles = (int)min((int64_t)kt_cta, KT - kt0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tid = lane & 3;
  const int64_t strip0 = ((int64_t)bx * 8 + warp) * kStripsPerWarp;
  const uint4* src = lay + (strip0 * KT + kt0) * 32 + lane;
  const int64_t b = (int64_t)kc * nbx + bx;
  const int64_t col0 = kt0 * 128;
  const uint4 Z = make_uint4(0, 0, 0, 0);
  int acc[kStripsPerWarp][4];
  // Three register buffers per strip, rotated by the 3x unrolled main loop:
  // tiles t and t + 1 in flight while tile t is consumed (kDepth = 2).
  uint4 bA[kStripsPerWarp], bB[kStripsPerWarp], bC[kStripsPerWarp];
  const uint4* nxt[kStripsPerWarp];  // next tile to prefetch, per strip
  pdl_trigger();  // the reduce kernel may be scheduled once every CTA has started
#pragma unroll
  for (int r = 0; r < kStripsPerWarp; ++r) {
    acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0;
    const uint4* p = src + r * KT * 32;
    bA[r] = ktiles > 0 ? ld_stream(p) : Z;
    bB[r] = ktiles > 1 ? ld_stream(p + 32) : Z;
    bC[r] = Z;
    nxt[r] = p + 32 * min(2, max(ktiles - 1, 0));
  }
  uint8_t* stage = reinterpret_cast<uint8_t*>(dg + kt_cta * 64);
  double* cvs = reinterpret_cast<double*>(stage + kOffBytes + 2 * kEntCap + 16);
#if GKB_BULK_STAGE
  // One thread stages the CTA's contiguous inputs with bulk copies on the TMA
  // engine, completing on one mbarrier: the block's list offsets (a 16-byte
  // aligned superset, oshift = the offsets' position in it) and list run
  // (immutable, before the PDL wait), then the range's correction
  // coefficients and digits (the predecessor's outputs, after it).
  // two mbarriers: [0] the digits (waited for before the loop), [1] the
  // epilogue's inputs (waited for after it, by each warp on its own)
  __shared__ __align__(8) uint64_t sbar[2];
  if (threadIdx.x == 0) {
    mbar_init(&sbar[0], 1);
    mbar_init(&sbar[1], 1);
  }
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(stage);
  int ent_shift = -1;
  int64_t eb = 0;
  uint32_t obytes = 0, ebytes = 0;
  const uint8_t* osrc = nullptr;
  const uint8_t* esrc = nullptr;
  if (m_off) {
    const uint32_t* orow = m_off + b * (kRowsPerCta + 1);
    osrc = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(orow) & ~uintptr_t(15));
    const uint32_t oshift = (uint32_t)(reinterpret_cast<const uint8_t*>(orow) - osrc);
    obytes = (oshift + 4 * (kRowsPerCta + 1) + 15) & ~15u;
    offs += oshift / 4;
    eb = m_base[b];
    const int64_t ne = orow[kRowsPerCta];
    const int64_t a0 = (eb * 2) & ~int64_t(15), a1 = (eb * 2 + ne * 2 + 15) & ~int64_t(15);
    if (a1 - a0 <= 2 * kEntCap) {
      esrc = reinterpret_cast<const uint8_t*>(m_ent) + a0;
      ebytes = (uint32_t)(a1 - a0);
      ent_shift = (int)(eb - a0 / 2);
    }
  }
  const int ncol = m_off ? (int)min((int64_t)ktiles * 128, C - col0) : 0;
  const double* csrc = cval + col0;
  // x may be a Krylov-basis column with an odd leading dimension: bulk only
  // when 16-byte aligned (an odd count's last element by a plain copy)
  const bool cbulk = m_off && ((reinterpret_cast<uintptr_t>(csrc) & 15) == 0);
  const uint32_t cbytes = cbulk ? (uint32_t)(ncol & ~1) * 8u : 0u;
  const uint32_t dbytes = (uint32_t)ktiles * 1024u;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&sbar[0], dbytes);
    mbar_arrive_expect_tx(&sbar[1], obytes + ebytes + cbytes);
    if (obytes) bulk_g2s(stage, osrc, obytes, &sbar[1]);
    if (ebytes) bulk_g2s(stage + kOffBytes, esrc, ebytes, &sbar[1]);
  }
  // everything above reads only the layout and the missing lists; from here
  // on the predecessor's outputs (digits, x / cm) are used
  pdl_wait();
  if (threadIdx.x == 0) {
    bulk_g2s(dg, dig + kt0 * 64, dbytes, &sbar[0]);
    if (cbytes) bulk_g2s(cvs, csrc, cbytes, &sbar[1]);
  }
  if (m_off && !cbulk) {
    for (int i = threadIdx.x; i < ncol; i += kThreads) cp_async8(cvs + i, csrc + i);
    cp_async_commit();
    cp_async_wait_all();
  } else if (cbulk && (ncol & 1) && threadIdx.x == kThreads - 1) {
    cvs[ncol - 1] = csrc[ncol - 1];
  }
  if (threadIdx.x == kThreads - 2) cvs[-1] = 0.0;  // walk_list_pair_u's zero slot (staging pad)
  __syncthreads();  // the mbarriers' init, the plain copies
  mbar_wait(&sbar[0], 0);
#else
  uint32_t* offs = reinterpret_cast<uint32_t*>(stage);
  // list entries: staged into shared memory (ent_shift = offset of the run's
  // first entry in the staged 16-byte-aligned copy), or -- a block denser in
  // missing entries than kEntCap -- walked in global memory (ent_shift < 0)
  int ent_shift = -1;
  int64_t eb = 0;
  if (m_off) {
    for (int i = threadIdx.x; i <= kRowsPerCta; i += kThreads)
      cp_async4(offs + i, m_off + b * (kRowsPerCta + 1) + i);
    eb = m_base[b];
    const int64_t ne = m_off[b * (kRowsPerCta + 1) + kRowsPerCta];
    const int64_t a0 = (eb * 2) & ~int64_t(15), a1 = (eb * 2 + ne * 2 + 15) & ~int64_t(15);
    if (a1 - a0 <= 2 * kEntCap) {
      const uint8_t* esrc = reinterpret_cast<const uint8_t*>(m_ent) + a0;
      for (int64_t i = threadIdx.x; i < (a1 - a0) / 16; i += kThreads)
        cp_async16(stage + kOffBytes + 16 * i, esrc + 16 * i);
      ent_shift = (int)(eb - a0 / 2);
    }
  }
  // everything above reads only the layout and the missing lists; from here
  // on the predecessor's outputs (digits, x / cm) are used
  pdl_wait();
  if (m_off) {
    // 8-byte copies: x may be a Krylov-basis column with an odd leading dimension
    const int ncol = (int)min((int64_t)ktiles * 128, C - col0);
    for (int i = threadIdx.x; i < ncol; i += kThreads) cp_async8(cvs + i, cval + col0 + i);
    cp_async_commit();
  }
  {
    const uint4* gd = dig + kt0 * 64;
    for (int i = threadIdx.x; i < ktiles * 64; i += kThreads) dg[i] = gd[i];
  }
#if GKB_EARLY_STAGE
  // the coefficient and list copies land together with the digits (both from
  // L2): one barrier, and each warp goes from its loop straight to its rows'
  // epilogue instead of waiting there for the CTA's slowest warp
  if (m_off) cp_async_wait_all();
#endif
  __syncthreads();
#endif
  // swizzled digit slots: the 8 lanes of each quarter-warp hit 8 distinct 16-byte bank groups
  const int sw = g ^ (2 * tid);
  const uint4* bp = dg + tid * 8 + sw;  // this thread's B fragments of tile t (64 uint4 per tile)
  // One tile: B fragments from shared memory, prefetch tile t + 2 into the
  // buffer freed by tile t - 1 (unconditional: past the last tile the pointer
  // stays on it, an L2 hit), MMAs on tile t.
#define GKB_PM_STEP(CUR, DST)                                              \
  if (t < ktiles) {                                                        \
    const uint4 b01 = bp[0], b23 = bp[32];                                 \
    const bool adv = t + 2 < ktiles - 1;                                   \
    const bool pf = kL2Pf > 0 && lane == 0 && t + kL2Pf < ktiles;          \
    _Pragma("unroll") for (int r = 0; r < kStripsPerWarp; ++r) {           \
      if (pf) prefetch_l2_512(nxt[r] + 32 * (kL2Pf - 2));                  \
      DST[r] = ld_stream(nxt[r]);                                          \
      nxt[r] += adv ? 32 : 0;                                              \
      mma_tile(acc[r], CUR[r], b01, b23);                                  \
    }                                                                      \
    bp += 64;                                                              \
    ++t;                                                                   \
  }
  if (ktiles == kFullRange) {
    // a full range: trip count known at compile time, fully unrolled -- no
    // per-tile bound test, clamp or counter; prefetch offsets are constants
    const uint4* p0 = src;
    const uint4* p1 = src + KT * 32;
#define GKB_PM_FULL(T, CUR, DST)                                           \
    {                                                                      \
      const uint4 b01 = bp[(T) * 64], b23 = bp[(T) * 64 + 32];             \
      if ((T) + 2 < kFullRange) {                                          \
        DST[0] = ld_stream(p0 + ((T) + 2) * 32);                           \
        if (kStripsPerWarp > 1) DST[kStripsPerWarp - 1] = ld_stream(p1 + ((T) + 2) * 32); \
      }                                                                    \
      _Pragma("unroll") for (int r = 0; r < kStripsPerWarp; ++r)           \
        mma_tile(acc[r], CUR[r], b01, b23);                                \
    }
#pragma unroll
    for (int T = 0; T < kFullRange; T += 3) {
      GKB_PM_FULL(T, bA, bC)
      if (T + 1 < kFullRange) GKB_PM_FULL(T + 1, bB, bA)
      if (T + 2 < kFullRange) GKB_PM_FULL(T + 2, bC, bB)
    }
#undef GKB_PM_FULL
  } else {
    for (int t = 0; t < ktiles;) {
      GKB_PM_STEP(bA, bC)
      GKB_PM_STEP(bB, bA)
      GKB_PM_STEP(bC, bB)
    }
  }
#undef GKB_PM_STEP
#if !GKB_EARLY_STAGE && !GKB_BULK_STAGE
  if (m_off) {
    cp_async_wait_all();
    __syncthreads();
  }
#endif
#if GKB_BULK_STAGE
  mbar_wait(&sbar[1], 0);  // the list run, offsets and coefficients
#endif
  // Epilogue. Thread (g, tid) holds digits (2 tid, 2 tid + 1) of rows g and
  // g + 8; 2^(16 tid) (D_2tid + 256 D_2tid+1) is exact in fp64, and the four
  // threads of the group add their parts by a butterfly (identical bits in
  // all four). Rows: tid 0/2 -> row g, tid 1/3 -> row g + 8; the two threads
  // of a row each walk half of its missing list.
  const int E = dexp[kc];
  const double rsum = dsum[kc];
  const double p0 = pow2(16 * tid), p1 = pow2(16 * tid + 8);
  double val[kStripsPerWarp], corr[kStripsPerWarp];
  int64_t rowr[kStripsPerWarp];
  uint32_t k0[kStripsPerWarp], ke[kStripsPerWarp];
#pragma unroll
  for (int r = 0; r < kStripsPerWarp; ++r) {
    double v0 = (double)acc[r][0] * p0 + (double)acc[r][1] * p1;
    double v1 = (double)acc[r][2] * p0 + (double)acc[r][3] * p1;
    v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
    v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
    v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
    v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
    const int hi = tid & 1;
    rowr[r] = (strip0 + r) * 16 + g + 8 * hi;
    val[r] = scale2(hi ? v1 : v0, E - 62);
    corr[r] = 0.0;
    if (m_off) {
      const int rl = (int)(rowr[r] - (int64_t)bx * kRowsPerCta);
      const uint32_t e0 = offs[rl], e1 = offs[rl + 1], mid = e0 + (e1 - e0) / 2;
      k0[r] = (tid >> 1) ? mid : e0;
      ke[r] = (tid >> 1) ? e1 : mid;
    }
  }
  if (m_off) {
    if (ent_shift >= 0) {  // shared-memory runs (pointer derived from the smem array: LDS)
      const uint16_t* ent = reinterpret_cast<const uint16_t*>(stage + kOffBytes) + ent_shift;
      if (kStripsPerWarp == 2)  // both strips' runs walked together (latencies overlap)
        walk_list_pair_u(ent, k0[0], ke[0], k0[kStripsPerWarp - 1], ke[kStripsPerWarp - 1], cvs,
                         corr[0], corr[kStripsPerWarp - 1]);
      else
#pragma unroll
        for (int r = 0; r < kStripsPerWarp; ++r) corr[r] = walk_list_u(ent, k0[r], ke[r], cvs);
    } else {
#pragma unroll
      for (int r = 0; r < kStripsPerWarp; ++r) corr[r] = walk_list_u(m_ent + eb, k0[r], ke[r], cvs);
    }
#pragma unroll
    for (int r = 0; r < kStripsPerWarp; ++r)  // both halves, commutative -> same bits
      corr[r] += __shfl_xor_sync(0xffffffffu, corr[r], 2);
  }
#pragma unroll
  for (int r = 0; r < kStripsPerWarp; ++r) {
    if ((tid >> 1) == 0) {
      const int64_t row = rowr[r];
      double out;
      if (MODE == 0) {  // a missing entry holds the imputed mean (genio.cpp:144)
        out = val[r] - mu[row] * rsum - (3.0 - mean[row]) * corr[r];
      } else {
        out = val[r] - rsum - corr[r];
      }
      part[(int64_t)kc * rows_pad + row] = out;
    }
  }
  if (tick) {  // K1 finish fused: the last range CTA of this row block sums the ranges in order
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(tick + bx, 1u) == (unsigned)(nkc - 1);
    __syncthreads();
    if (last) {
      __threadfence();
      for (int jr = threadIdx.x; jr < kRowsPerCta; jr += kThreads) {
        const int64_t j = (int64_t)bx * kRowsPerCta + jr;
        if (j < R) {
          double a = 0.0;
          for (int c = 0; c < nkc; ++c) a += __ldcg(part + (int64_t)c * rows_pad + j);
          yout[j] = inv_s[j] * a;  // (may be a page-locked host buffer: one write per row)
        }
      }
      if (threadIdx.x == 0) tick[bx] = 0u;
    }
  }
}


// ---------------------------------------------------------------- single-layout mode
// K2 (reference apply_adjoint, z = X^T y) read from layout 1 (rows = SNPs),
// for shards whose two layouts do not fit in HBM (config 5 at 2 GPUs: 125 GB
// per layout per GPU). The contraction runs over SNPs, but a layout-1 word
// holds 16 samples of ONE SNP, so a lane first gathers 4 SNPs' words of the
// same 16 samples (two 8-byte loads from the tile's fragment order) and
// byte-transposes them (8 PRMT): z_b byte i = SNP i's 4 codes of samples
// 4b..4b+3. The shift-free mask z_b & (0x03030303 << 2q) is then a
// register of 4 SNPs (k) for ONE sample (4b + q) scaled by 4^q, i.e. an A
// fragment of mma.m16n8k16 (k-group = the lane's 4 SNPs, rows = samples).
// The 4^q scale is per output row and undone exactly in the epilogue. Per
// 512-byte tile: 2 LDG.64, 8 PRMT, 16 LOP3, 8 IMMA (vs 4 IMMA + 16 LOP3 in
// the two-layout kernel). CTA = 8 warps x one 128-sample tile column each
// (1024 samples) x a range of 112 SNP strips (1792 SNPs); per lane 8
// accumulator sets (16 samples x 2 digits).
constexpr int kL1tStrips = 112;               // SNP strips per range (1792 SNPs)
constexpr int kL1tRows = 1024;                // samples per CTA
constexpr int kL1tOffBytes = ((kL1tRows + 1) * 4 + 15) / 16 * 16;
constexpr int kL1tEntBytes = 40 * 1024;       // staged list bytes (longer: walked in global)
size_t l1t_smem_bytes() {
  return (size_t)kL1tStrips * 128 + (size_t)kL1tStrips * 16 * 8 + kL1tOffBytes + kL1tEntBytes + 16;
}

__device__ __forceinline__ void mma16_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ uint2 ld_stream8(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p));
  return v;
}

// two strips (A, B) of one tile column: per strip, words w (SNPs 2t, 2t+8 of
// word-column g) and v (SNPs 2t+1, 2t+9); strip A is the MMA's k-group t and
// strip B the k-group 4 + t of mma.m16n8k32 (bd: digit g of both)
__device__ __forceinline__ void l1t_transpose(const uint2 w, const uint2 v, uint32_t (&z)[4]) {
  // k order i = 0..3 <-> SNPs 2t, 2t+1, 2t+8, 2t+9 (k_digitize<2>'s positions)
  const uint32_t t0 = prmt(w.x, v.x, 0x5140u), t1 = prmt(w.x, v.x, 0x7362u);
  const uint32_t t2 = prmt(w.y, v.y, 0x5140u), t3 = prmt(w.y, v.y, 0x7362u);
  z[0] = prmt(t0, t2, 0x5410u);
  z[1] = prmt(t0, t2, 0x7632u);
  z[2] = prmt(t1, t3, 0x5410u);
  z[3] = prmt(t1, t3, 0x7632u);
}
__device__ __forceinline__ void mma_tile_l1t(int (&acc)[8][4], const uint2 wa, const uint2 va,
                                             const uint2 wb, const uint2 vb, const uint32_t bda,
                                             const uint32_t bdb) {
  uint32_t za[4], zb[4];
  l1t_transpose(wa, va, za);
  l1t_transpose(wb, vb, zb);
  const uint32_t m0 = 0x03030303u, m1 = m0 << 2, m2 = m0 << 4, m3 = m0 << 6;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    // samples 4b, 4b+1 (x1, x4) and 4b+2, 4b+3 (x16, x64); rows g / g + 8
    mma_u8s8(acc[2 * b], za[b] & m0, za[b] & m1, zb[b] & m0, zb[b] & m1, bda, bdb);
    mma_u8s8(acc[2 * b + 1], za[b] & m2, za[b] & m3, zb[b] & m2, zb[b] & m3, bda, bdb);
  }
}

// grid (sample blocks, SNP ranges). Writes part[kc][sample] = the range's
// exact partial of z_s = sum_j c_j a_js - sum_j c_j mu_j - sum_{j miss} cm_j.
#ifndef GKB_L1T_MINB
#define GKB_L1T_MINB 2  // CTAs per SM (register budget of the strip-pair loop)
#endif
__global__ void __launch_bounds__(kThreads, GKB_L1T_MINB) k_pm_adj_l1(
    const uint32_t* __restrict__ lay, int64_t KT, int64_t S1, const uint32_t* __restrict__ dig,
    const int* __restrict__ dexp, const double* __restrict__ dsum,
    const double* __restrict__ cval, const uint32_t* __restrict__ m_off,
    const int64_t* __restrict__ m_base, const uint16_t* __restrict__ m_ent, int64_t rows_pad,
    double* __restrict__ part) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* dgs = reinterpret_cast<uint32_t*>(sm);                      // 112 strips x 32 words
  double* cvs = reinterpret_cast<double*>(sm + kL1tStrips * 128);        // 1792 cm values
  uint8_t* stage = sm + kL1tStrips * 128 + kL1tStrips * 16 * 8;          // offsets, then entries
  const int kc = blockIdx.y, bx = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t kt = (int64_t)bx * 8 + warp;
  const bool live = kt < KT;
  const int64_t s0 = (int64_t)kc * kL1tStrips;
  const int ns = (int)min((int64_t)kL1tStrips, S1 - s0);
  const int64_t b = (int64_t)kc * gridDim.x + bx;
  // this lane's two 8-byte halves of the tile (fragment order, word_index):
  // uint4 #(8t + (g & 3)) and #(8t + 4 + (g & 3)), half g >> 2
  const uint2* lay2 = reinterpret_cast<const uint2*>(lay);
  const int64_t o1 = (int64_t)(8 * t + (g & 3)) * 2 + (g >> 2), o2 = o1 + 8;
  const uint2* pw = lay2 + ((s0 * KT + (live ? kt : 0)) * 32) * 2 + o1;
  const int64_t sstride = KT * 64;  // uint2 per strip
  int acc[8][4];
#pragma unroll
  for (int m = 0; m < 8; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0;
  const uint2 Z = make_uint2(0, 0);
  // strip pairs (s, s + 1): a pair's second strip beyond the layout rereads
  // the first (its digits are zero: rows >= p_loc)
  const int np = (ns + 1) / 2;
  const int64_t d12 = o2 - o1;
  auto pair_ptr = [&](int q) { return pw + sstride * (2 * (int64_t)q); };
  auto second = [&](int q) { return 2 * q + 1 < ns ? sstride : 0; };
  uint2 aw0 = Z, av0 = Z, bw0 = Z, bv0 = Z, aw1 = Z, av1 = Z, bw1 = Z, bv1 = Z;
  if (np > 0) {
    const uint2* p = pair_ptr(0);
    aw0 = ld_stream8(p);
    av0 = ld_stream8(p + d12);
    bw0 = ld_stream8(p + second(0));
    bv0 = ld_stream8(p + second(0) + d12);
  }
  if (np > 1) {
    const uint2* p = pair_ptr(1);
    aw1 = ld_stream8(p);
    av1 = ld_stream8(p + d12);
    bw1 = ld_stream8(p + second(1));
    bv1 = ld_stream8(p + second(1) + d12);
  }
  uint2 aw2 = Z, av2 = Z, bw2 = Z, bv2 = Z;
  pdl_trigger();
  __shared__ __align__(8) uint64_t sbar[2];
  if (threadIdx.x == 0) {
    mbar_init(&sbar[0], 1);
    mbar_init(&sbar[1], 1);
  }
  // staging: offsets (aligned superset) + list run before the PDL wait,
  // digits (barrier 0) and cm values (barrier 1) after it
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(stage);
  int ent_shift = -1;
  int64_t eb = 0;
  uint32_t obytes = 0, ebytes = 0;
  const uint8_t* osrc = nullptr;
  const uint8_t* esrc = nullptr;
  if (m_off) {
    const uint32_t* orow = m_off + b * (kL1tRows + 1);
    osrc = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(orow) & ~uintptr_t(15));
    const uint32_t oshift = (uint32_t)(reinterpret_cast<const uint8_t*>(orow) - osrc);
    obytes = (oshift + 4 * (kL1tRows + 1) + 15) & ~15u;
    offs += oshift / 4;
    eb = m_base[b];
    const int64_t ne = orow[kL1tRows];
    const int64_t a0 = (eb * 2) & ~int64_t(15), a1 = (eb * 2 + ne * 2 + 15) & ~int64_t(15);
    if (a1 - a0 <= kL1tEntBytes) {
      esrc = reinterpret_cast<const uint8_t*>(m_ent) + a0;
      ebytes = (uint32_t)(a1 - a0);
      ent_shift = (int)(eb - a0 / 2);
    }
  }
  const uint32_t dbytes = (uint32_t)kL1tStrips * 128u;
  const uint32_t cbytes = m_off ? (uint32_t)kL1tStrips * 16u * 8u : 0u;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&sbar[0], dbytes);
    mbar_arrive_expect_tx(&sbar[1], obytes + ebytes + cbytes);
    if (obytes) bulk_g2s(stage, osrc, obytes, &sbar[1]);
    if (ebytes) bulk_g2s(stage + kL1tOffBytes, esrc, ebytes, &sbar[1]);
  }
  pdl_wait();
  if (threadIdx.x == 0) {
    bulk_g2s(dgs, dig + (int64_t)kc * kL1tStrips * 32, dbytes, &sbar[0]);
    if (cbytes) bulk_g2s(cvs, cval + (int64_t)kc * kL1tStrips * 16, cbytes, &sbar[1]);
  }
  __syncthreads();  // the mbarriers' init
  mbar_wait(&sbar[0], 0);
  const uint32_t* bq = dgs + g * 4 + t;  // digit g of the lane's k-group, strip by strip
  // pair q in buffer (q mod 3); pair q + 2 prefetched into the buffer of q - 1
#define GKB_L1T_STEP(AW, AV, BW, BV, NAW, NAV, NBW, NBV)                   \
  if (q < np) {                                                            \
    const uint32_t bda = bq[64 * q], bdb = bq[64 * q + 32];                \
    if (q + 2 < np) {                                                      \
      const uint2* p = pair_ptr(q + 2);                                    \
      NAW = ld_stream8(p);                                                 \
      NAV = ld_stream8(p + d12);                                           \
      NBW = ld_stream8(p + second(q + 2));                                 \
      NBV = ld_stream8(p + second(q + 2) + d12);                           \
    }                                                                      \
    mma_tile_l1t(acc, AW, AV, BW, BV, bda, bdb);                           \
    ++q;                                                                   \
  }
  for (int q = 0; q < np;) {
    GKB_L1T_STEP(aw0, av0, bw0, bv0, aw2, av2, bw2, bv2)
    GKB_L1T_STEP(aw1, av1, bw1, bv1, aw0, av0, bw0, bv0)
    GKB_L1T_STEP(aw2, av2, bw2, bv2, aw1, av1, bw1, bv1)
  }
#undef GKB_L1T_STEP
  mbar_wait(&sbar[1], 0);  // offsets, list run, cm values
  // Epilogue. Lane (g, t) holds digits (2t, 2t+1) of 16 samples of word-column
  // g: MMA 2b + h -> rows g / g + 8 = samples 4b + 2h / 4b + 2h + 1. A
  // reduce-scatter over the 4 lanes of the group (xor 1, then xor 2: the tree
  // of the two-layout kernel's butterfly) leaves lane t the sums of samples
  // 4t..4t+3 (q = 0..3).
  const double p0 = pow2(16 * t), p1 = pow2(16 * t + 8);
  double V[4][4];
#pragma unroll
  for (int bb = 0; bb < 4; ++bb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      V[bb][2 * h] = (double)acc[2 * bb + h][0] * p0 + (double)acc[2 * bb + h][1] * p1;
      V[bb][2 * h + 1] = (double)acc[2 * bb + h][2] * p0 + (double)acc[2 * bb + h][3] * p1;
    }
  double W[2][4];
  const bool odd = t & 1;
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double keep = odd ? V[2 * k + 1][q] : V[2 * k][q];
      const double send = odd ? V[2 * k][q] : V[2 * k + 1][q];
      W[k][q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
  double S[4];
  const bool hi2 = t & 2;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double keep = hi2 ? W[1][q] : W[0][q];
    const double send = hi2 ? W[0][q] : W[1][q];
    S[q] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  if (!live) return;
  const int E = dexp[kc];
  const double rsum = dsum[kc];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rl = warp * 128 + 16 * g + 4 * t + q;  // block-local sample row
    double corr = 0.0;
    if (m_off) {
      const uint32_t e0 = offs[rl], e1 = offs[rl + 1];
      corr = ent_shift >= 0
                 ? walk_list_u(reinterpret_cast<const uint16_t*>(stage + kL1tOffBytes) + ent_shift,
                             e0, e1, cvs)
                 : walk_list_u(m_ent + eb, e0, e1, cvs);
    }
    const double val = scale2(S[q], E - 62 - 2 * q);
    part[(int64_t)kc * rows_pad + (int64_t)bx * kL1tRows + rl] = val - rsum - corr;
  }
}

// Missing lists of the single-layout K2 blocks (1024 samples x 1792 SNPs),
// read from layout 1: thread per sample row; entries = block-local SNP
// indices (ascending). Count pass / fill pass as k_miss_tiles.
template <bool kFill>
__global__ void __launch_bounds__(kL1tRows) k_miss_l1t(const uint32_t* __restrict__ lay,
                                                     int64_t KT, int64_t p_loc, int64_t n,
                                                     uint32_t* __restrict__ cnt,
                                                     const uint32_t* __restrict__ off,
                                                     const int64_t* __restrict__ base,
                                                     uint16_t* __restrict__ ent) {
  const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int r = threadIdx.x;
  const int64_t smp = (int64_t)blockIdx.x * kL1tRows + r;
  const int64_t j0 = (int64_t)blockIdx.y * kL1tStrips * 16;
  const int64_t j1 = min(p_loc, j0 + (int64_t)kL1tStrips * 16);
  uint32_t c = 0;
  int64_t pos = kFill ? base[b] + off[b * (kL1tRows + 1) + r] : 0;
  if (smp < n) {
    const int64_t wc = smp >> 4;
    const int sh = 2 * (int)(smp & 15);
    for (int64_t j = j0; j < j1; ++j) {
      const uint32_t code = (lay[word_index(KT, j, wc)] >> sh) & 3u;
      if (code == 3u) {
        if (kFill) ent[pos++] = (uint16_t)(j - j0);
        else ++c;
      }
    }
  }
  if (!kFill) cnt[b * kL1tRows + r] = c;
}

// CTA per block: exclusive scan of 1024 row counts -> off, block total -> tot.
__global__ void __launch_bounds__(kL1tRows) k_block_scan_1024(const uint32_t* __restrict__ cnt,
                                                            uint32_t* __restrict__ off,
                                                            int64_t* __restrict__ tot) {
  __shared__ uint32_t sc[kL1tRows];
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  sc[t] = cnt[b * kL1tRows + t];
  __syncthreads();
  for (int o = 1; o < kL1tRows; o <<= 1) {
    const uint32_t v = t >= o ? sc[t - o] : 0u;
    __syncthreads();
    sc[t] += v;
    __syncthreads();
  }
  if (t == 0) off[b * (kL1tRows + 1)] = 0;
  off[b * (kL1tRows + 1) + t + 1] = sc[t];
  if (t == kL1tRows - 1) tot[b] = sc[t];
}

// ---------------------------------------------------------------- dense-missing mode
// Main kernel for shards with many missing entries (DESIGN.md section 4,
// "Missing data"): no lists. The missing indicator of a word, t = w & (w >> 1)
// & 0x5555... (code 3 = missing), is expanded exactly like the codes (one LOP3
// per fragment register: 0 or 4^q per byte) and multiplied on the tensor
// cores with a digit set into a second exact accumulator:
//   K1 (MODE 0): the same digits (of x): corr_j = sum_{s miss} x_s,
//                y_j = inv_s_j (val_j - mu_j X - (3 - m_j) corr_j);
//   K2 (MODE 1): the digits of cm_j = c_j (3 - m_j) (dig2):
//                z_s = val_s - sum_j c_j mu_j - sum_{j miss} cm_j.
// Both corrections are exact integer sums scaled like the main sum (the
// list walk's fp64 sums are replaced by exact ones), and the kernel's cost
// does not depend on the missing rate.
__device__ __forceinline__ uint4 miss_ind(const uint4 w) {
  uint4 t;
  t.x = w.x & (w.x >> 1) & 0x55555555u;
  t.y = w.y & (w.y >> 1) & 0x55555555u;
  t.z = w.z & (w.z >> 1) & 0x55555555u;
  t.w = w.w & (w.w >> 1) & 0x55555555u;
  return t;
}

// mma_tile of the missing indicators of w: the group-q register is
// w & (w >> 1) & (0x01010101 << 2q) -- one shift per word and one LOP3 per
// register (the same values as miss_ind(w) & (0x03030303 << 2q))
__device__ __forceinline__ uint32_t and3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;  // one LOP3 (the compiler would share a & b and spend two per register)
  asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ void mma_tile_ind(int (&acc)[4], const uint4 w, const uint4 b01,
                                             const uint4 b23) {
  const uint32_t m0 = 0x01010101u, m1 = m0 << 2, m2 = m0 << 4, m3 = m0 << 6;
  const uint32_t sx = w.x >> 1, sy = w.y >> 1, sz = w.z >> 1, sw = w.w >> 1;
  mma_u8s8(acc, and3(w.x, sx, m0), and3(w.y, sy, m0), and3(w.x, sx, m1), and3(w.y, sy, m1),
           b01.x, b01.y);
  mma_u8s8(acc, and3(w.x, sx, m2), and3(w.y, sy, m2), and3(w.x, sx, m3), and3(w.y, sy, m3),
           b01.z, b01.w);
  mma_u8s8(acc, and3(w.z, sz, m0), and3(w.w, sw, m0), and3(w.z, sz, m1), and3(w.w, sw, m1),
           b23.x, b23.y);
  mma_u8s8(acc, and3(w.z, sz, m2), and3(w.w, sw, m2), and3(w.z, sz, m3), and3(w.w, sw, m3),
           b23.z, b23.w);
}

size_t pmi_smem_bytes(int kt_cta, int mode) {
  return (size_t)kt_cta * 64 * 16 * (mode ? 2 : 1);
}

template <int MODE>
// CTAs per SM: K1 fits 64 registers (4), K2's second digit set does not (3)
__global__ void __launch_bounds__(kThreads, MODE == 0 ? 4 : 3) k_pm_ind(
    const uint4* __restrict__ lay, int64_t KT, int kt_cta, const uint4* __restrict__ dig,
    const int* __restrict__ dexp, const double* __restrict__ dsum,
    const uint4* __restrict__ dig2, const int* __restrict__ dexp2,
    const double* __restrict__ mu, const double* __restrict__ mean, int64_t rows_pad,
    double* __restrict__ part) {
  extern __shared__ __align__(16) uint4 dg[];  // kt_cta * 64 digits [, K2: kt_cta * 64 of cm]
  const int kc = blockIdx.y, bx = blockIdx.x;
  const int64_t kt0 = (int64_t)kc * kt_cta;
  const int ktiles = (int)min((int64_t)kt_cta, KT - kt0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tid = lane & 3;
  const int64_t strip0 = ((int64_t)bx * 8 + warp) * kStripsPerWarp;
  const uint4* src = lay + (strip0 * KT + kt0) * 32 + lane;
  const uint4 Z = make_uint4(0, 0, 0, 0);
  int acc[kStripsPerWarp][4], accm[kStripsPerWarp][4];
  uint4 bA[kStripsPerWarp], bB[kStripsPerWarp], bC[kStripsPerWarp];
  const uint4* nxt[kStripsPerWarp];
  pdl_trigger();
#pragma unroll
  for (int r = 0; r < kStripsPerWarp; ++r) {
    acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0;
    accm[r][0] = accm[r][1] = accm[r][2] = accm[r][3] = 0;
    const uint4* p = src + r * KT * 32;
    bA[r] = ktiles > 0 ? ld_stream(p) : Z;
    bB[r] = ktiles > 1 ? ld_stream(p + 32) : Z;
    bC[r] = Z;
    nxt[r] = p + 32 * min(2, max(ktiles - 1, 0));
  }
  __shared__ __align__(8) uint64_t sbar;
  if (threadIdx.x == 0) mbar_init(&sbar, 1);
  const uint32_t dbytes = (uint32_t)ktiles * 1024u;
  pdl_wait();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&sbar, MODE ? 2 * dbytes : dbytes);
    bulk_g2s(dg, dig + kt0 * 64, dbytes, &sbar);
    if (MODE) bulk_g2s(dg + kt_cta * 64, dig2 + kt0 * 64, dbytes, &sbar);
  }
  __syncthreads();  // the mbarrier's init
  mbar_wait(&sbar, 0);
  const int sw = g ^ (2 * tid);
  const uint4* bp = dg + tid * 8 + sw;
  const int m2 = MODE ? kt_cta * 64 : 0;  // K2: the cm digits' offset
#define GKB_PMI_STEP(CUR, DST)                                             \
  if (t < ktiles) {                                                        \
    const uint4 b01 = bp[0], b23 = bp[32];                                 \
    const uint4 c01 = MODE ? bp[m2] : b01, c23 = MODE ? bp[m2 + 32] : b23; \
    const bool adv = t + 2 < ktiles - 1;                                   \
    _Pragma("unroll") for (int r = 0; r < kStripsPerWarp; ++r) {           \
      DST[r] = ld_stream(nxt[r]);                                          \
      nxt[r] += adv ? 32 : 0;                                              \
      mma_tile(acc[r], CUR[r], b01, b23);                                  \
      mma_tile_ind(accm[r], CUR[r], c01, c23);                       \
    }                                                                      \
    bp += 64;                                                              \
    ++t;                                                                   \
  }
  if (ktiles == kFullRange) {
    // a full range: fully unrolled, constant prefetch offsets (as k_pm_main)
    const uint4* p0 = src;
    const uint4* p1 = src + KT * 32;
#define GKB_PMI_FULL(T, CUR, DST)                                          \
    {                                                                      \
      const uint4 b01 = bp[(T) * 64], b23 = bp[(T) * 64 + 32];             \
      const uint4 c01 = MODE ? bp[(T) * 64 + m2] : b01;                    \
      const uint4 c23 = MODE ? bp[(T) * 64 + m2 + 32] : b23;               \
      if ((T) + 2 < kFullRange) {                                          \
        DST[0] = ld_stream(p0 + ((T) + 2) * 32);                           \
        DST[kStripsPerWarp - 1] = ld_stream(p1 + ((T) + 2) * 32);          \
      }                                                                    \
      _Pragma("unroll") for (int r = 0; r < kStripsPerWarp; ++r) {         \
        mma_tile(acc[r], CUR[r], b01, b23);                                \
        mma_tile_ind(accm[r], CUR[r], c01, c23);                     \
      }                                                                    \
    }
    static_assert(kStripsPerWarp == 2, "the unrolled loop prefetches strips 0 and 1");
#pragma unroll
    for (int T = 0; T < kFullRange; T += 3) {
      GKB_PMI_FULL(T, bA, bC)
      if (T + 1 < kFullRange) GKB_PMI_FULL(T + 1, bB, bA)
      if (T + 2 < kFullRange) GKB_PMI_FULL(T + 2, bC, bB)
    }
#undef GKB_PMI_FULL
  } else {
    for (int t = 0; t < ktiles;) {
      GKB_PMI_STEP(bA, bC)
      GKB_PMI_STEP(bB, bA)
      GKB_PMI_STEP(bC, bB)
    }
  }
#undef GKB_PMI_STEP
  const int E = dexp[kc], Em = MODE ? dexp2[kc] : E;
  const double rsum = dsum[kc];
  const double p0 = pow2(16 * tid), p1 = pow2(16 * tid + 8);
  const int hi = tid & 1;
#pragma unroll
  for (int r = 0; r < kStripsPerWarp; ++r) {
    double v0 = (double)acc[r][0] * p0 + (double)acc[r][1] * p1;
    double v1 = (double)acc[r][2] * p0 + (double)acc[r][3] * p1;
    double u0 = (double)accm[r][0] * p0 + (double)accm[r][1] * p1;
    double u1 = (double)accm[r][2] * p0 + (double)accm[r][3] * p1;
    v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
    v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
    v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
    v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
    u0 += __shfl_xor_sync(0xffffffffu, u0, 1);
    u0 += __shfl_xor_sync(0xffffffffu, u0, 2);
    u1 += __shfl_xor_sync(0xffffffffu, u1, 1);
    u1 += __shfl_xor_sync(0xffffffffu, u1, 2);
    if ((tid >> 1) == 0) {
      const int64_t row = (strip0 + r) * 16 + g + 8 * hi;
      const double val = scale2(hi ? v1 : v0, E - 62);
      const double cor = scale2(hi ? u1 : u0, Em - 62);
      double out;
      if (MODE == 0) {  // a missing entry holds the imputed mean (genio.cpp:144)
        out = val - mu[row] * rsum - (3.0 - mean[row]) * cor;
      } else {
        out = val - rsum - cor;
      }
      part[(int64_t)kc * rows_pad + row] = out;
    }
  }
}

// ---------------------------------------------------------------- two vectors per pass
// Block products ("decode amortized over k"): the same
// kernel for two coefficient vectors at once. Each tile is loaded and expanded
// once; every group of four A registers feeds one MMA per vector. Digits,
// integer sums, the epilogue and the list walk are the single-vector kernel's,
// in the same order, so each column equals its single-vector product bit for
// bit. 3 CTAs/SM (two digit sets and two coefficient stagings in shared memory).
struct PM2Args {
  const uint4* dig[2];
  const int* dexp[2];
  const double* dsum[2];
  const double* cval[2];
  double* part[2];
};

__device__ __forceinline__ void mma_tile2(int (&a0)[4], int (&a1)[4], const uint4 w,
                                          const uint4 b01a, const uint4 b23a, const uint4 b01b,
                                          const uint4 b23b) {
  const uint32_t m0 = 0x03030303u, m1 = m0 << 2, m2 = m0 << 4, m3 = m0 << 6;
  uint32_t p0 = w.x & m0, p1 = w.y & m0, p2 = w.x & m1, p3 = w.y & m1;
  mma_u8s8(a0, p0, p1, p2, p3, b01a.x, b01a.y);
  mma_u8s8(a1, p0, p1, p2, p3, b01b.x, b01b.y);
  p0 = w.x & m2; p1 = w.y & m2; p2 = w.x & m3; p3 = w.y & m3;
  mma_u8s8(a0, p0, p1, p2, p3, b01a.z, b01a.w);
  mma_u8s8(a1, p0, p1, p2, p3, b01b.z, b01b.w);
  p0 = w.z & m0; p1 = w.w & m0; p2 = w.z & m1; p3 = w.w & m1;
  mma_u8s8(a0, p0, p1, p2, p3, b23a.x, b23a.y);
  mma_u8s8(a1, p0, p1, p2, p3, b23b.x, b23b.y);
  p0 = w.z & m2; p1 = w.w & m2; p2 = w.z & m3; p3 = w.w & m3;
  mma_u8s8(a0, p0, p1, p2, p3, b23a.z, b23a.w);
  mma_u8s8(a1, p0, p1, p2, p3, b23b.z, b23b.w);
}

// walk_list2 in one predicated chunk loop (as walk_list_u; same bits)
__device__ __forceinline__ void walk_list2_u(const uint16_t* __restrict__ ent, uint32_t k0,
                                             uint32_t ke, const double* __restrict__ cva,
                                             const double* __restrict__ cvb, double& ca,
                                             double& cb) {
  double sa = 0.0, sb = 0.0;
  const uint32_t n = ke - k0;
#pragma unroll 1
  for (uint32_t i = 0; i < n; i += 4) {
    double x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u < n) {
        const int c = ent[k0 + i + u];
        x[u] = cva[c];
        y[u] = cvb[c];
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u < n) sa += x[u];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u < n) sb += y[u];
  }
  ca = sa;
  cb = sb;
}

size_t pm2_smem_bytes(int kt_cta) {
  return 2 * (size_t)kt_cta * 64 * 16 + kOffBytes + 2 * kEntCap + 16 + 2 * (size_t)kt_cta * 128 * 8;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 3) k_pm_main2(
    const uint4* __restrict__ lay, int64_t KT, int kt_cta, PM2Args a,
    const double* __restrict__ mu, const double* __restrict__ mean,
    const uint32_t* __restrict__ m_off, const int64_t* __restrict__ m_base,
    const uint16_t* __restrict__ m_ent, int64_t rows_pad, int64_t C) {
  extern __shared__ __align__(16) uint4 dg[];  // 2 x kt_cta * 64 digits, then list staging
  const int kc = blockIdx.y;
  const int64_t kt0 = (int64_t)kc * kt_cta;
  const int ktiles = (int)min((int64_t)kt_cta, KT - kt0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tid = lane & 3;
  const int64_t strip0 = ((int64_t)blockIdx.x * 8 + warp) * kStripsPerWarp;
  const uint4* src = lay + (strip0 * KT + kt0) * 32 + lane;
  const int64_t b = (int64_t)kc * gridDim.x + blockIdx.x;
  const int64_t col0 = kt0 * 128;
  const uint4 Z = make_uint4(0, 0, 0, 0);
  int acc0[kStripsPerWarp][4], acc1[kStripsPerWarp][4];
  uint4 bA[kStripsPerWarp], bB[kStripsPerWarp], bC[kStripsPerWarp];
  const uint4* nxt[kStripsPerWarp];
  pdl_trigger();
#pragma unroll
  for (int r = 0; r < kStripsPerWarp; ++r) {
    acc0[r][0] = acc0[r][1] = acc0[r][2] = acc0[r][3] = 0;
    acc1[r][0] = acc1[r][1] = acc1[r][2] = acc1[r][3] = 0;
    const uint4* p = src + r * KT * 32;
    bA[r] = ktiles > 0 ? ld_stream(p) : Z;
    bB[r] = ktiles > 1 ? ld_stream(p + 32) : Z;
    bC[r] = Z;
    nxt[r] = p + 32 * min(2, max(ktiles - 1, 0));
  }
  uint4* dg1 = dg + kt_cta * 64;
  uint8_t* stage = reinterpret_cast<uint8_t*>(dg + 2 * kt_cta * 64);
  double* cvs0 = reinterpret_cast<double*>(stage + kOffBytes + 2 * kEntCap + 16);
  double* cvs1 = cvs0 + kt_cta * 128;
#if GKB_BULK_STAGE
  // bulk-copy staging on one mbarrier, as in k_pm_main (two digit sets and
  // two coefficient vectors)
  __shared__ __align__(8) uint64_t sbar;
  if (threadIdx.x == 0) mbar_init(&sbar, 1);
  const uint32_t* offs = reinterpret_cast<const uint32_t*>(stage);
  int ent_shift = -1;
  int64_t eb = 0;
  uint32_t obytes = 0, ebytes = 0;
  const uint8_t* osrc = nullptr;
  const uint8_t* esrc = nullptr;
  if (m_off) {
    const uint32_t* orow = m_off + b * (kRowsPerCta + 1);
    osrc = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(orow) & ~uintptr_t(15));
    const uint32_t oshift = (uint32_t)(reinterpret_cast<const uint8_t*>(orow) - osrc);
    obytes = (oshift + 4 * (kRowsPerCta + 1) + 15) & ~15u;
    offs += oshift / 4;
    eb = m_base[b];
    const int64_t ne = orow[kRowsPerCta];
    const int64_t a0 = (eb * 2) & ~int64_t(15), a1 = (eb * 2 + ne * 2 + 15) & ~int64_t(15);
    if (a1 - a0 <= 2 * kEntCap) {
      esrc = reinterpret_cast<const uint8_t*>(m_ent) + a0;
      ebytes = (uint32_t)(a1 - a0);
      ent_shift = (int)(eb - a0 / 2);
    }
  }
  const int ncol = m_off ? (int)min((int64_t)ktiles * 128, C - col0) : 0;
  const double* csrc0 = a.cval[0] + col0;
  const double* csrc1 = a.cval[1] + col0;
  const bool cbulk = m_off && ((reinterpret_cast<uintptr_t>(csrc0) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(csrc1) & 15) == 0);
  const uint32_t cbytes = cbulk ? (uint32_t)(ncol & ~1) * 8u : 0u;
  const uint32_t dbytes = (uint32_t)ktiles * 1024u;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&sbar, obytes + ebytes + 2 * cbytes + 2 * dbytes);
    if (obytes) bulk_g2s(stage, osrc, obytes, &sbar);
    if (ebytes) bulk_g2s(stage + kOffBytes, esrc, ebytes, &sbar);
  }
  pdl_wait();
  if (threadIdx.x == 0) {
    if (cbytes) {
      bulk_g2s(cvs0, csrc0, cbytes, &sbar);
      bulk_g2s(cvs1, csrc1, cbytes, &sbar);
    }
    bulk_g2s(dg, a.dig[0] + kt0 * 64, dbytes, &sbar);
    bulk_g2s(dg1, a.dig[1] + kt0 * 64, dbytes, &sbar);
  }
  if (m_off && !cbulk) {
    for (int i = threadIdx.x; i < ncol; i += kThreads) {
      cp_async8(cvs0 + i, csrc0 + i);
      cp_async8(cvs1 + i, csrc1 + i);
    }
    cp_async_commit();
    cp_async_wait_all();
  } else if (cbulk && (ncol & 1) && threadIdx.x == kThreads - 1) {
    cvs0[ncol - 1] = csrc0[ncol - 1];
    cvs1[ncol - 1] = csrc1[ncol - 1];
  }
  __syncthreads();  // the mbarrier's init, the plain copies
  mbar_wait(&sbar, 0);
#else
  uint32_t* offs = reinterpret_cast<uint32_t*>(stage);
  int ent_shift = -1;
  int64_t eb = 0;
  if (m_off) {
    for (int i = threadIdx.x; i <= kRowsPerCta; i += kThreads)
      cp_async4(offs + i, m_off + b * (kRowsPerCta + 1) + i);
    eb = m_base[b];
    const int64_t ne = m_off[b * (kRowsPerCta + 1) + kRowsPerCta];
    const int64_t a0 = (eb * 2) & ~int64_t(15), a1 = (eb * 2 + ne * 2 + 15) & ~int64_t(15);
    if (a1 - a0 <= 2 * kEntCap) {
      const uint8_t* esrc = reinterpret_cast<const uint8_t*>(m_ent) + a0;
      for (int64_t i = threadIdx.x; i < (a1 - a0) / 16; i += kThreads)
        cp_async16(stage + kOffBytes + 16 * i, esrc + 16 * i);
      ent_shift = (int)(eb - a0 / 2);
    }
  }
  pdl_wait();
  if (m_off) {
    const int ncol = (int)min((int64_t)ktiles * 128, C - col0);
    for (int i = threadIdx.x; i < ncol; i += kThreads) {
      cp_async8(cvs0 + i, a.cval[0] + col0 + i);
      cp_async8(cvs1 + i, a.cval[1] + col0 + i);
    }
    cp_async_commit();
  }
  {
    const uint4* gd0 = a.dig[0] + kt0 * 64;
    const uint4* gd1 = a.dig[1] + kt0 * 64;
    for (int i = threadIdx.x; i < ktiles * 64; i += kThreads) {
      dg[i] = gd0[i];
      dg1[i] = gd1[i];
    }
  }
#if GKB_EARLY_STAGE
  if (m_off) cp_async_wait_all();  // as in k_pm_main
#endif
  __syncthreads();
#endif
  const int sw = g ^ (2 * tid);
  const uint4* bp = dg + tid * 8 + sw;
#define GKB_PM2_STEP(CUR, DST)                                             \
  if (t < ktiles) {                                                        \
    const uint4 b01a = bp[0], b23a = bp[32];                               \
    const uint4 b01b = bp[kt_cta * 64], b23b = bp[kt_cta * 64 + 32];       \
    const bool adv = t + 2 < ktiles - 1;                                   \
    _Pragma("unroll") for (int r = 0; r < kStripsPerWarp; ++r) {           \
      DST[r] = ld_stream(nxt[r]);                                          \
      nxt[r] += adv ? 32 : 0;                                              \
      mma_tile2(acc0[r], acc1[r], CUR[r], b01a, b23a, b01b, b23b);         \
    }                                                                      \
    bp += 64;                                                              \
    ++t;                                                                   \
  }
  for (int t = 0; t < ktiles;) {
    GKB_PM2_STEP(bA, bC)
    GKB_PM2_STEP(bB, bA)
    GKB_PM2_STEP(bC, bB)
  }
#undef GKB_PM2_STEP
#if !GKB_EARLY_STAGE && !GKB_BULK_STAGE
  if (m_off) {
    cp_async_wait_all();
    __syncthreads();
  }
#endif
  const int E0 = a.dexp[0][kc], E1 = a.dexp[1][kc];
  const double rs0 = a.dsum[0][kc], rs1 = a.dsum[1][kc];
  const double p0 = pow2(16 * tid), p1 = pow2(16 * tid + 8);
#pragma unroll
  for (int r = 0; r < kStripsPerWarp; ++r) {
    double u0 = (double)acc0[r][0] * p0 + (double)acc0[r][1] * p1;
    double u1 = (double)acc0[r][2] * p0 + (double)acc0[r][3] * p1;
    double v0 = (double)acc1[r][0] * p0 + (double)acc1[r][1] * p1;
    double v1 = (double)acc1[r][2] * p0 + (double)acc1[r][3] * p1;
    u0 += __shfl_xor_sync(0xffffffffu, u0, 1);
    u0 += __shfl_xor_sync(0xffffffffu, u0, 2);
    u1 += __shfl_xor_sync(0xffffffffu, u1, 1);
    u1 += __shfl_xor_sync(0xffffffffu, u1, 2);
    v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
    v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
    v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
    v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
    const int hi = tid & 1;
    const int64_t row = (strip0 + r) * 16 + g + 8 * hi;
    const int rl = (int)(row - (int64_t)blockIdx.x * kRowsPerCta);
    const double val0 = scale2(hi ? u1 : u0, E0 - 62);
    const double val1 = scale2(hi ? v1 : v0, E1 - 62);
    double c0 = 0.0, c1 = 0.0;
    if (m_off) {
      const uint32_t e0 = offs[rl], e1 = offs[rl + 1], mid = e0 + (e1 - e0) / 2;
      const uint32_t k0 = (tid >> 1) ? mid : e0, ke = (tid >> 1) ? e1 : mid;
      if (ent_shift >= 0)
        walk_list2_u(reinterpret_cast<const uint16_t*>(stage + kOffBytes) + ent_shift, k0, ke,
                     cvs0, cvs1, c0, c1);
      else
        walk_list2_u(m_ent + eb, k0, ke, cvs0, cvs1, c0, c1);
      c0 += __shfl_xor_sync(0xffffffffu, c0, 2);
      c1 += __shfl_xor_sync(0xffffffffu, c1, 2);
    }
    if ((tid >> 1) == 0) {
      double o0, o1;
      if (MODE == 0) {
        o0 = val0 - mu[row] * rs0 - (3.0 - mean[row]) * c0;
        o1 = val1 - mu[row] * rs1 - (3.0 - mean[row]) * c1;
      } else {
        o0 = val0 - rs0 - c0;
        o1 = val1 - rs1 - c1;
      }
      a.part[0][(int64_t)kc * rows_pad + row] = o0;
      a.part[1][(int64_t)kc * rows_pad + row] = o1;
    }
  }
}

// ---------------------------------------------------------------- tcgen05 block products
// Block products of k >= 3 coefficient vectors in ONE pass over the layout
// (VERDICT r1 item 9): the 5th-generation tensor cores (tcgen05.mma
// kind::i8, SASS UTCIMMA) with the accumulators in tensor memory. CTA = 256
// rows (two M = 128 accumulators) x one column range (kt_cta tiles); per
// tile the 8 warps expand their strips' 2-bit codes AND missing indicators
// (w & (w >> 1) & 0x55..) to u8 in shared memory (the shift-free masks, one
// 16-byte K chunk per word, canonical K-major no-swizzle layout), one thread
// bulk-copies the tile's B image (digits of all k vectors: N = 8k rows) and
// issues 16 MMAs (4 K-steps x codes / indicators x two row halves),
// committed to the buffer's "empty" mbarrier (2 buffers). TMEM columns:
// [0, N) codes rows 0-127, [N, 2N) codes rows 128-255, [2N, 3N) and
// [3N, 4N) the indicators. The missing corrections are exact integer sums
// (no lists): K1 (MODE 0) multiplies the indicators with the same digits
// (sum_{s miss} x_s); K2 (MODE 1) with the digits of cm_j = c_j (3 - m_j)
// (a second B image). Epilogue: tcgen05.ld per row; the row value is
// sum_i D_i 256^i 2^(E - 62) as in the mma.sync kernels.
constexpr int kTcRows = 256;
__device__ __forceinline__ void umma_i8(uint32_t dt, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// smem A / B images: canonical K-major with the 128-byte swizzle (atoms of
// 8 rows x 128 B, 1024-byte aligned; row r's 16-byte chunk c at
// (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) * 16)): one tile's K
// (128 bytes per row) is one atom row, and the producers' quarter-warps
// store to 8 distinct bank groups
__device__ __host__ __forceinline__ uint32_t tc_sw_off(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t addr) {
  uint64_t d = (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;           // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset: 8-row atoms
  d |= (uint64_t)1 << 46;            // sm_100 descriptor version
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

size_t tc_smem_bytes(int k, int mode) {
  const size_t N = 8 * (size_t)k;
  // 2 buffers x (codes + indicators (2 x 32 KB) + B image(s) N x 128 B), 1 KB alignment slack
  return 2 * (2 * 32768 + N * 128 * (mode ? 2 : 1)) + 1024;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads + 32, 1) k_pm_blk_tc(
    const uint4* __restrict__ lay, int64_t KT, int kt_cta, int k, int kpad,
    const uint8_t* __restrict__ tdig, const uint8_t* __restrict__ tdig2,
    const int* __restrict__ dexp, const int* __restrict__ dexp2, const double* __restrict__ dsum,
    const double* __restrict__ mu, const double* __restrict__ mean, int64_t rows_pad, int nkc,
    double* __restrict__ part) {
  extern __shared__ __align__(16) uint8_t tsm[];  // aligned to 1024 below
  // N = 8 kpad: kpad = k rounded up to even (N a multiple of 16: kind::i8 at
  // M = 128 raised an illegal instruction for N = 40, 56, ... on this part)
  const int N = 8 * kpad;
  const uint32_t bimg = (uint32_t)N * 128u;  // B image bytes per tile
  // buffer: [codes h0 | codes h1 | ind h0 | ind h1] (16 KB each), B [, B2]
  const uint32_t bufsz = 65536u + bimg * (MODE ? 2u : 1u);
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tsm) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t fullb[2], emptyb[2];
  __shared__ uint32_t tbase;
  const int kc = blockIdx.y, bx = blockIdx.x;
  const int64_t kt0 = (int64_t)kc * kt_cta;
  const int ktiles = (int)min((int64_t)kt_cta, KT - kt0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool mma_warp = warp == 8;  // warps 0-7 produce, warp 8 issues the MMAs
  uint32_t ncols = 32;
  while (ncols < 4u * (uint32_t)N) ncols <<= 1;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&fullb[b], 8 + 1);  // 8 producer warps + the B bulk copy's arrival
      mbar_init(&emptyb[b], 1);     // the MMA commit
    }
  }
  if (mma_warp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  pdl_wait();  // the digits are the predecessor's output
  if (mma_warp) {
    if (lane == 0) {
      // kind::i8 instruction descriptor: D s32, A u8, B s8, K-major, N, M = 128
      const uint32_t idesc = (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
      for (int t = 0; t < ktiles; ++t) {
        const int b = t & 1;
        mbar_wait(&fullb[b], (uint32_t)((t >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(base + (size_t)b * bufsz), sb = sa + 65536;
        const uint32_t sb2 = sb + (MODE ? bimg : 0u);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // K = 32 bytes per MMA: 32 B into the atom rows
          const uint32_t acc = (t > 0 || ks > 0) ? 1u : 0u;
          const uint64_t db = umma_desc_sw128(sb + ks * 32);
          const uint64_t dbm = umma_desc_sw128(sb2 + ks * 32);
          umma_i8(tmem, umma_desc_sw128(sa + ks * 32), db, idesc, acc);
          umma_i8(tmem + (uint32_t)N, umma_desc_sw128(sa + 16384 + ks * 32), db, idesc, acc);
          umma_i8(tmem + 2u * (uint32_t)N, umma_desc_sw128(sa + 32768 + ks * 32), dbm, idesc,
                  acc);
          umma_i8(tmem + 3u * (uint32_t)N, umma_desc_sw128(sa + 49152 + ks * 32), dbm, idesc,
                  acc);
        }
        umma_commit(&emptyb[b]);
      }
    }
    __syncwarp();
  } else {
    const int g = lane >> 2, tid = lane & 3;
    const int64_t strip0 = ((int64_t)bx * 8 + warp) * 2;  // this warp's two strips
    const uint4* src0 = lay + (strip0 * KT + kt0) * 32 + lane;
    const uint4* src1 = src0 + KT * 32;
    const uint32_t m0 = 0x03030303u, m1 = m0 << 2, m2 = m0 << 4, m3 = m0 << 6;
    const uint4 Z = make_uint4(0, 0, 0, 0);
    // three register buffers: tiles t + 1 and t + 2 in flight while t is stored
    uint4 pa0 = ktiles > 0 ? ld_stream(src0) : Z, pa1 = ktiles > 0 ? ld_stream(src1) : Z;
    uint4 pb0 = ktiles > 1 ? ld_stream(src0 + 32) : Z, pb1 = ktiles > 1 ? ld_stream(src1 + 32) : Z;
    uint4 pc0 = Z, pc1 = Z;
    const int half = warp >> 2;      // rows 0-127 / 128-255
    const int r0 = (warp & 3) * 32;  // this warp's first row in its half
    const int sw = (g & 1) ? 2 : 0;  // odd rows store their c + 4 chunks first: 8 bank groups
    auto stage = [&](int t, const uint4& c0, const uint4& c1) {
      const int b = t & 1;
      uint8_t* buf = base + (size_t)b * bufsz;
      // the MMAs of tile t - 2 must have released this buffer
      if (t >= 2) mbar_wait(&emptyb[b], (uint32_t)(((t >> 1) - 1) & 1));
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&fullb[b], bimg * (MODE ? 2u : 1u));
        const size_t toff = ((size_t)kc * kt_cta + t) * bimg;
        bulk_g2s(buf + 65536, tdig + toff, bimg, &fullb[b]);
        if (MODE) bulk_g2s(buf + 65536 + bimg, tdig2 + toff, bimg, &fullb[b]);
      }
      // lane (g, tid) holds words (row g, col tid), (g + 8, tid), (g, tid + 4),
      // (g + 8, tid + 4) of each strip; one 16-byte K chunk per word
#pragma unroll
      for (int sidx = 0; sidx < 2; ++sidx) {
        const uint4 w = sidx ? c1 : c0;
        // words j = (row g, col tid), (g + 8, tid), (g, tid + 4), (g + 8, tid + 4),
        // taken in the order jj ^ sw (selects, no local-memory array)
        const uint32_t lo0 = sw ? w.z : w.x, lo1 = sw ? w.w : w.y;
        const uint32_t hi0 = sw ? w.x : w.z, hi1 = sw ? w.y : w.w;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = jj ^ sw;
          const int r = r0 + 16 * sidx + g + 8 * (j & 1), c = tid + 4 * (j >> 1);
          const uint32_t x = jj == 0 ? lo0 : jj == 1 ? lo1 : jj == 2 ? hi0 : hi1;
          const uint32_t mi = x & (x >> 1) & 0x55555555u;
          const uint32_t off = tc_sw_off(r, c);
          *reinterpret_cast<uint4*>(buf + half * 16384 + off) =
              make_uint4(x & m0, x & m1, x & m2, x & m3);
          *reinterpret_cast<uint4*>(buf + 32768 + half * 16384 + off) =
              make_uint4(mi & m0, mi & m1, mi & m2, mi & m3);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // STS -> tensor core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&fullb[b]);
    };
    for (int t = 0; t < ktiles;) {
#define GKB_TC_STEP(C0, C1, N0, N1)                                       \
      if (t < ktiles) {                                                   \
        if (t + 2 < ktiles) {                                             \
          N0 = ld_stream(src0 + 32 * (t + 2));                            \
          N1 = ld_stream(src1 + 32 * (t + 2));                            \
        }                                                                 \
        stage(t, C0, C1);                                                 \
        ++t;                                                              \
      }
      GKB_TC_STEP(pa0, pa1, pc0, pc1)
      GKB_TC_STEP(pb0, pb1, pa0, pa1)
      GKB_TC_STEP(pc0, pc1, pb0, pb1)
#undef GKB_TC_STEP
    }
  }
  // every MMA done AND every commit arrival landed before this CTA's shared
  // memory can be reused: wait for the last completion of both "empty"
  // barriers (an unwaited asynchronous arrival would hit the next CTA's smem)
  if (ktiles >= 1) mbar_wait(&emptyb[(ktiles - 1) & 1], (uint32_t)(((ktiles - 1) >> 1) & 1));
  if (ktiles >= 2) mbar_wait(&emptyb[(ktiles - 2) & 1], (uint32_t)(((ktiles - 2) >> 1) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (!mma_warp) {
    // epilogue: warp w reads TMEM lanes 32 (w & 3) .. + 31 of its half
    const int half = warp >> 2, r0 = (warp & 3) * 32;
    const int64_t row = (int64_t)bx * kTcRows + half * 128 + r0 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const double rmu = MODE == 0 ? mu[row] : 0.0, rmean = MODE == 0 ? mean[row] : 0.0;
    for (int v = 0; v < k; ++v) {
      uint32_t dc[8], dm[8];
      tmem_ld8(lanebase + (uint32_t)(half * N + 8 * v), dc);
      tmem_ld8(lanebase + (uint32_t)(2 * N + half * N + 8 * v), dm);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // sum_i D_i 256^i: per 16-bit pair exact, pairs added in digit order
      double vc = 0.0, vm = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        vc += ((double)(int)dc[2 * i] + 256.0 * (double)(int)dc[2 * i + 1]) * pow2(16 * i);
        vm += ((double)(int)dm[2 * i] + 256.0 * (double)(int)dm[2 * i + 1]) * pow2(16 * i);
      }
      const int E = dexp[(int64_t)v * nkc + kc];
      const double val = scale2(vc, E - 62);
      double out;
      if (MODE == 0) {
        const double cor = scale2(vm, E - 62);
        out = val - rmu * dsum[(int64_t)v * nkc + kc] - (3.0 - rmean) * cor;
      } else {
        const double cor = scale2(vm, dexp2[(int64_t)v * nkc + kc] - 62);
        out = val - dsum[(int64_t)v * nkc + kc] - cor;
      }
      part[((int64_t)v * nkc + kc) * rows_pad + row] = out;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (mma_warp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols)
                 : "memory");
}

// Digits of k vectors for k_pm_blk_tc, one CTA per (span, vector): the B
// image of each tile (N = 8 kpad rows x 128 K bytes, 128-byte swizzle): row
// 8v + i, chunk wc (the tile's word column), byte 4q + e <-> column
// 16 wc + 4e + q (the shift-free masks' byte order) with the 4^-q group
// prescale. MODE 0: v = x; MODE 1: v = inv_s y (dsum = sum v mu), and the
// digits of cm = v (3 - mean) into dig2 (exponent dexp2). A vector's 1 KB of
// each tile is staged in shared memory and written out with 16-byte stores.
constexpr int kTcSpan = 56;  // tiles per span (7168 columns): |D| <= 192 x 127 x 7168 < 2^31
template <int MODE>
__global__ void __launch_bounds__(1024) k_digitize_tc(const double* __restrict__ X, int64_t ldx,
                                                      int k, const double* __restrict__ inv_s,
                                                      const double* __restrict__ mu,
                                                      const double* __restrict__ mean, int64_t C,
                                                      int kt_cta, uint8_t* __restrict__ dig,
                                                      uint8_t* __restrict__ dig2,
                                                      int* __restrict__ dexp,
                                                      int* __restrict__ dexp2,
                                                      double* __restrict__ dsum) {
  extern __shared__ __align__(16) uint8_t dsh[];  // kt_cta KB [, MODE 1: + kt_cta KB]
  __shared__ double red[33];
  __shared__ int redi[33];
  pdl_wait();
  pdl_trigger();
  const int kc = blockIdx.x, v = blockIdx.y, nkc = gridDim.x;
  const int N = 8 * gridDim.y;  // gridDim.y = kpad; vectors v >= k are zero
  const bool pad = v >= k;
  const int ncol = kt_cta * 128;
  const int64_t c0 = (int64_t)kc * ncol;
  const double* xin = X + (int64_t)(pad ? 0 : v) * ldx;
  int emax = -1100, emax2 = -1100;
  double psum = 0.0;
  for (int t = threadIdx.x; t < ncol; t += blockDim.x) {
    const int64_t c = c0 + t;
    if (c < C && !pad) {
      double val = xin[c];
      if (MODE == 1) {
        val = inv_s[c] * val;
        psum += val * mu[c];
        emax2 = max(emax2, exp_of(val * (3.0 - mean[c])));
      } else {
        psum += val;
      }
      emax = max(emax, exp_of(val));
    }
  }
  const int E = block_max_int(emax, redi);
  const int E2 = MODE ? block_max_int(emax2, redi) : 0;
  const double sm = block_sum(psum, red);
  uint8_t* sd2 = dsh + (size_t)kt_cta * 1024;
  for (int t = threadIdx.x; t < ncol; t += blockDim.x) {
    const int64_t c = c0 + t;
    double val = 0.0, cmv = 0.0;
    if (c < C && !pad) {
      val = xin[c];
      if (MODE == 1) {
        val = inv_s[c] * val;
        cmv = val * (3.0 - mean[c]);
      }
    }
    const int tile = t >> 7, wc = (t >> 4) & 7, k16 = t & 15, q = k16 & 3, e = k16 >> 2;
    // rows 8v + i of the tile's B image (128-byte swizzle, tc_sw_off): this
    // vector's 1 KB block of the tile, staged
    const int off0 = tile * 1024 + 4 * q + e;
    long long M = __double2ll_rn(scale2(val, 62 - E - 2 * q));
    long long M2 = MODE ? __double2ll_rn(scale2(cmv, 62 - E2 - 2 * q)) : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int off = off0 + i * 128 + ((wc ^ i) << 4);
      const int d = (int)(signed char)(M & 0xFF);
      M = (M - d) >> 8;
      dsh[off] = (uint8_t)d;
      if (MODE) {
        const int d2 = (int)(signed char)(M2 & 0xFF);
        M2 = (M2 - d2) >> 8;
        sd2[off] = (uint8_t)d2;
      }
    }
  }
  __syncthreads();
  for (int u = threadIdx.x; u < kt_cta * 64; u += blockDim.x) {  // 16-byte units
    const int tile = u >> 6, w = u & 63;
    const size_t dst = ((size_t)kc * kt_cta + tile) * (size_t)N * 128 + (size_t)v * 1024 + 16 * w;
    *reinterpret_cast<uint4*>(dig + dst) = reinterpret_cast<const uint4*>(dsh)[u];
    if (MODE) *reinterpret_cast<uint4*>(dig2 + dst) = reinterpret_cast<const uint4*>(sd2)[u];
  }
  if (threadIdx.x == 0 && !pad) {
    dexp[(int64_t)v * nkc + kc] = E;
    dsum[(int64_t)v * nkc + kc] = sm;
    if (MODE) dexp2[(int64_t)v * nkc + kc] = E2;
  }
}

// ---------------------------------------------------------------- marker scan
// Per-marker fits y ~ [1, m_i, Z] (regress.cpp:10-65 per marker, by
// Frisch-Waugh-Lovell -- paper_1808_03374_b200/regress.py): one thread per
// marker i reads P[i, :] = [m_i.y, m_i.C] of the block product, the marker's
// counts and scaling, and the shared nuisance algebra (A^-1 = (C'C)^-1, w = C'y,
// y'y - w'A^-1 w), and writes beta, se, intercept, sigma2 and the dependency flag.
__global__ void k_marker_scan(const double* __restrict__ P, int64_t ldp, int64_t rows, int K,
                              const double* __restrict__ Ainv, const double* __restrict__ w,
                              double yyc, double a0w, double denom,
                              const int64_t* __restrict__ counts, const double* __restrict__ mu,
                              const double* __restrict__ inv_s, const double* __restrict__ mean,
                              double* __restrict__ beta, double* __restrict__ se,
                              double* __restrict__ icpt, double* __restrict__ sig2,
                              int* __restrict__ dep) {
  extern __shared__ double ms[];  // Ainv (K x K) then w (K)
  pdl_wait();
  pdl_trigger();
  for (int t = threadIdx.x; t < K * K + K; t += blockDim.x) ms[t] = t < K * K ? Ainv[t] : w[t - K * K];
  __syncthreads();
  const double* Ai = ms;
  const double* ws = ms + K * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* c = counts + 4 * i;
    const double m = mu[i], is = inv_s[i], mn = mean[i];
    const double q = ((double)c[0] * m * m + (double)c[1] * (1.0 - m) * (1.0 - m) +
                      (double)c[2] * (2.0 - m) * (2.0 - m) + (double)c[3] * (mn - m) * (mn - m)) *
                     (is * is);
    double my = P[i], d = q, uw = 0.0, au0 = 0.0;
    for (int a = 0; a < K; ++a) {  // AU_a = sum_b u_b Ainv[b, a];  d -= AU_a u_a
      double au = 0.0;
      for (int b = 0; b < K; ++b) au += P[(int64_t)(1 + b) * ldp + i] * Ai[b + a * K];
      if (a == 0) au0 = au;
      d -= au * P[(int64_t)(1 + a) * ldp + i];
      uw += au * ws[a];
    }
    const int distinct = (c[0] > 0) + (c[1] > 0) + (c[2] > 0);
    const double bt = (my - uw) / d;
    const double rss = yyc - bt * bt * d;
    const double s2 = rss / denom;
    beta[i] = bt;
    sig2[i] = s2;
    se[i] = sqrt(s2 / d);
    icpt[i] = a0w - bt * au0;
    dep[i] = (distinct < 2 || is == 0.0 || !(d > 0.0)) ? 1 : 0;
  }
}

// K1 finish: y_j = inv_s_j * sum_kc part[kc][j] (ranges in order)
__global__ void k1_reduce(const double* __restrict__ part, int nkc, int64_t rows_pad,
                          int64_t p_loc, const double* __restrict__ inv_s,
                          double* __restrict__ y) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  if (j >= p_loc) return;
  const double* p = part + j;
  double acc = 0.0;
  int c = 0;
  for (; c + 8 <= nkc; c += 8) {  // 8 loads in flight, added in range order
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldcs(p + (int64_t)(c + i) * rows_pad);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i];
  }
  for (; c < nkc; ++c) acc += __ldcs(p + (int64_t)c * rows_pad);
  y[j] = inv_s[j] * acc;
}

// K2 finish: z_s = sum_kc part[kc][s]. Block = 32 warps x 32 consecutive
// samples: warp w sums ranges kc = w (mod 32) with lanes on consecutive
// samples (coalesced); partials added in warp order -> deterministic.
__global__ void __launch_bounds__(1024) k2_reduce(const double* __restrict__ part, int nkc,
                                                  int64_t rows_pad, int64_t n,
                                                  double* __restrict__ z) {
  __shared__ double ps[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s = (int64_t)blockIdx.x * 32 + lane;
  pdl_wait();
  double acc = 0.0;
  if (s < n)
#pragma unroll 4
    for (int c = warp; c < nkc; c += 32) acc += part[(int64_t)c * rows_pad + s];
  ps[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && s < n) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += ps[w][lane];
    z[s] = t;
  }
}

// K2 finish for tall sample counts (n >= kK2SeqMin): thread per sample, the
// ranges in order (as k1_reduce), 8 coalesced loads in flight per thread.
// The 32-warp block above keeps short vectors spread over the SMs; here there
// are enough samples, and its one-or-two loads per thread with a block
// barrier ran at ~2.2 TB/s on config 4 (n = 500,000: 224 MB of partials).
constexpr int64_t kK2SeqMin = 65536;
__global__ void __launch_bounds__(256) k2_reduce_seq(const double* __restrict__ part, int nkc,
                                                     int64_t rows_pad, int64_t n,
                                                     double* __restrict__ z) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  if (s >= n) return;
  const double* p = part + s;
  double acc = 0.0;
  int c = 0;
  for (; c + 8 <= nkc; c += 8) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldcs(p + (int64_t)(c + i) * rows_pad);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i];
  }
  for (; c < nkc; ++c) acc += __ldcs(p + (int64_t)c * rows_pad);
  z[s] = acc;
}

// every K2 finish (two-layout, single-layout, block products) goes through
// here, so a given (n, nkc) always sums its partials in the same order
void launch_k2_reduce(const double* part, int nkc, int64_t rows_pad, int64_t n, double* z,
                      cudaStream_t s) {
  if (n >= kK2SeqMin)
    launch_pdl(k2_reduce_seq, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, true, part, nkc,
               rows_pad, n, z);
  else
    launch_pdl(k2_reduce, dim3((unsigned)((n + 31) / 32)), dim3(1024), 0, s, true, part, nkc,
               rows_pad, n, z);
}

int grid_for(int64_t work, int threads, int cap = 148 * 16) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

// ---------------------------------------------------------------- host side
PMPlan pm_plan(int64_t R, int64_t C) {
  PMPlan pl;
  pl.R = R;
  pl.C = C;
  pl.S = ((R + 15) / 16 + kStripsPerCta - 1) / kStripsPerCta * kStripsPerCta;  // whole CTAs
  if (pl.S < kStripsPerCta) pl.S = kStripsPerCta;
  pl.KT = (C + 127) / 128;
  if (pl.KT < 1) pl.KT = 1;
  pl.kt_cta = kFullRange;  // 1792 columns per CTA (14 KB of digits); 12-20 swept, 14 best (config 2 and 3)
  if (const char* e = std::getenv("GKB_KT_CTA")) pl.kt_cta = std::max(1, std::atoi(e));  // sweeps
  pl.nkc = (int)((pl.KT + pl.kt_cta - 1) / pl.kt_cta);
  pl.grid_x = pl.S / kStripsPerCta;
  pl.rows_cta = kRowsPerCta;
  pl.rows_pad = pl.S * 16;
  pl.smem = pm_smem_bytes(pl.kt_cta);
  pl.dig_smem = (size_t)pl.kt_cta * 64 * sizeof(uint4) + (size_t)pl.kt_cta * 128 * sizeof(double);
  return pl;
}

int64_t pm_words(const PMPlan& pl) { return pl.S * pl.KT * 128; }

void build_lt1(const uint8_t* bed, int64_t stride_bytes, int64_t rows, int64_t row0, int64_t n,
               const PMPlan& pl, uint32_t* lay, cudaStream_t s) {
  const int64_t W = (n + 15) / 16;
  if (rows * W == 0) return;
  k_build_lt1<<<grid_for(rows * W, 256), 256, 0, s>>>(bed, stride_bytes, rows, row0, n, W, pl.KT,
                                                      lay);
}

void build_lt2(const uint8_t* bed, int64_t stride_bytes, int64_t rows, int64_t row0, int64_t n,
               const PMPlan& pl, uint32_t* lay, cudaStream_t s) {
  const int64_t W = (n + 15) / 16;
  const int64_t work = ((rows + 15) / 16) * W;
  if (work == 0) return;
  k_build_lt2<<<grid_for(work, 128), 128, 0, s>>>(bed, stride_bytes, rows, row0, n, W, pl.KT, lay);
}

void marker_counts(const uint32_t* lay1, const PMPlan& pl1, int64_t p_loc, int64_t n,
                   int64_t* counts, cudaStream_t s) {
  if (p_loc == 0) return;
  k_marker_counts<<<grid_for(p_loc * 32, 256), 256, 0, s>>>(lay1, pl1.KT, p_loc, (n + 15) / 16, n,
                                                             counts);
}

void layout_to_bed(const uint32_t* lay1, const PMPlan& pl1, int64_t n, int64_t row0,
                   int64_t nrows, uint8_t* out, cudaStream_t s) {
  const int64_t work = nrows * ((n + 15) / 16);
  if (work == 0) return;
  k_layout_to_bed<<<grid_for(work, 256), 256, 0, s>>>(lay1, pl1.KT, n, row0, nrows, out);
}

void miss_lists(const uint32_t* lay, const PMPlan& pl, bool fill, uint32_t* cnt,
                const uint32_t* off, const int64_t* base, uint16_t* ent, cudaStream_t s) {
  dim3 grid((unsigned)pl.grid_x, (unsigned)pl.nkc);
  if (fill)
    k_miss_tiles<true><<<grid, kRowsPerCta, 0, s>>>(lay, pl.KT, pl.kt_cta, cnt, off, base, ent);
  else
    k_miss_tiles<false><<<grid, kRowsPerCta, 0, s>>>(lay, pl.KT, pl.kt_cta, cnt, off, base, ent);
}

void block_scan(const uint32_t* cnt, int64_t nblk, int span, uint32_t* off, int64_t* tot,
                cudaStream_t s) {
  if (nblk == 0) return;
  k_block_scan<<<(unsigned)nblk, 512, 0, s>>>(cnt, span, off, tot);
}

L1TPlan l1t_plan(const PMPlan& pl1, int64_t p_loc) {
  L1TPlan lt;
  lt.grid_x = (pl1.KT + 7) / 8;  // 8 tiles (1024 samples) per CTA
  lt.nkc = std::max<int64_t>(1, (p_loc + kL1tStrips * 16 - 1) / (kL1tStrips * 16));
  lt.rows_pad = lt.grid_x * kL1tRows;
  return lt;
}

size_t l1t_dig_bytes() { return (size_t)kL1tStrips * 128; }

void miss_lists_l1t(const uint32_t* lay1, const PMPlan& pl1, const L1TPlan& lt, int64_t p_loc,
                    int64_t n, bool fill, uint32_t* cnt, const uint32_t* off, const int64_t* base,
                    uint16_t* ent, cudaStream_t s) {
  dim3 grid((unsigned)lt.grid_x, (unsigned)lt.nkc);
  if (fill)
    k_miss_l1t<true><<<grid, kL1tRows, 0, s>>>(lay1, pl1.KT, p_loc, n, cnt, off, base, ent);
  else
    k_miss_l1t<false><<<grid, kL1tRows, 0, s>>>(lay1, pl1.KT, p_loc, n, cnt, off, base, ent);
}

void block_scan_1024(const uint32_t* cnt, int64_t nblk, uint32_t* off, int64_t* tot,
                     cudaStream_t s) {
  if (nblk == 0) return;
  k_block_scan_1024<<<(unsigned)nblk, kL1tRows, 0, s>>>(cnt, off, tot);
}

namespace {
template <class K>
void allow_smem(K kern, size_t bytes) {  // opt in above 48 KB
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
}  // namespace

void k1_digitize(const GenoView& g, const double* x, cudaStream_t s, const DivIn& di) {
  const PMPlan& pl = g.pl1;
  allow_smem(k_digitize<0>, pl.dig_smem);
  launch_pdl(k_digitize<0>, dim3((unsigned)pl.nkc), dim3(1024), pl.dig_smem, s, true, x,
             (const double*)nullptr, (const double*)nullptr, (const double*)nullptr, g.n, pl.kt_cta,
             g.s1.dig, g.s1.dexp, g.s1.dsum, (double*)nullptr, di.div, di.store, di.gate, (uint4*)nullptr, (int*)nullptr);
}

void k2_digitize(const GenoView& g, const double* y, cudaStream_t s, const DivIn& di) {
  const PMPlan& pl = g.pl2;
  // dense-missing mode: the cm digits (k_pm_ind's second digit set) in the same launch
  const size_t smem = g.ind ? 2 * pl.dig_smem : pl.dig_smem;
  allow_smem(k_digitize<1>, smem);
  launch_pdl(k_digitize<1>, dim3((unsigned)pl.nkc), dim3(1024), smem, s, true, y,
             (const double*)g.inv_s, (const double*)g.mu, (const double*)g.mean, g.p_loc,
             pl.kt_cta, g.s2.dig, g.s2.dexp, g.s2.dsum, g.s2.cm, di.div, di.store, di.gate,
             g.ind ? g.s2m.dig : (uint4*)nullptr, g.ind ? g.s2m.dexp : (int*)nullptr);
}

namespace {
template <int MODE>
void launch_main(const GenoView& g, const PMPlan& pl, const uint4* lay, const PMScratch& sc,
                 const double* cval, const MissLists& ml, cudaStream_t s, bool pdl,
                 double* fused_out = nullptr) {
  auto kern = k_pm_main<MODE>;
  allow_smem(kern, pl.smem);
  // fused K1 finish: grid (nkc, row blocks), ranges of a row block adjacent
  const bool fused = fused_out != nullptr;
  const dim3 grid = fused ? dim3((unsigned)pl.nkc, (unsigned)pl.grid_x)
                          : dim3((unsigned)pl.grid_x, (unsigned)pl.nkc);
  launch_pdl(kern, grid, dim3(kThreads), pl.smem, s, pdl, lay, pl.KT, pl.kt_cta,
             (const uint4*)sc.dig, (const int*)sc.dexp, (const double*)sc.dsum, cval,
             (const double*)g.mu, (const double*)g.mean, ml.off, ml.base, ml.ent, pl.rows_pad,
             pl.C, sc.part, fused ? sc.tick : (unsigned*)nullptr,
             (const double*)(fused ? g.inv_s : nullptr), fused_out, pl.R);
}
}  // namespace

namespace {
// dense-missing mode: no lists; K2 also needs the digits of cm (s2m)
template <int MODE>
void launch_ind(const GenoView& g, const PMPlan& pl, const uint4* lay, const PMScratch& sc,
                cudaStream_t s, bool pdl) {
  auto kern = k_pm_ind<MODE>;
  const size_t smem = pmi_smem_bytes(pl.kt_cta, MODE);
  allow_smem(kern, smem);
  launch_pdl(kern, dim3((unsigned)pl.grid_x, (unsigned)pl.nkc), dim3(kThreads), smem, s, pdl,
             lay, pl.KT, pl.kt_cta, (const uint4*)sc.dig, (const int*)sc.dexp,
             (const double*)sc.dsum, (const uint4*)g.s2m.dig, (const int*)g.s2m.dexp,
             (const double*)g.mu, (const double*)g.mean, pl.rows_pad, sc.part);
}
}  // namespace

namespace {
// single-layout mode: K2's digitize (digits in k_pm_adj_l1 order) and main kernel
void digitize_l1t(const GenoView& g, const double* y, cudaStream_t s, const DivIn& di) {
  const size_t smem = (size_t)14 * 64 * sizeof(uint4) + (size_t)14 * 128 * sizeof(double);
  allow_smem(k_digitize<2>, smem);
  launch_pdl(k_digitize<2>, dim3((unsigned)g.l1t_nkc), dim3(1024), smem, s, true, y,
             (const double*)g.inv_s, (const double*)g.mu, (const double*)g.mean, g.p_loc, 14,
             g.s2.dig, g.s2.dexp, g.s2.dsum, g.s2.cm, di.div, di.store, di.gate, (uint4*)nullptr, (int*)nullptr);
}
void launch_adj_l1(const GenoView& g, cudaStream_t s, bool pdl) {
  const size_t smem = l1t_smem_bytes();
  allow_smem(k_pm_adj_l1, smem);
  launch_pdl(k_pm_adj_l1, dim3((unsigned)g.l1t_grid, (unsigned)g.l1t_nkc), dim3(kThreads), smem,
             s, pdl, reinterpret_cast<const uint32_t*>(g.lt1), g.pl1.KT, g.pl1.S,
             reinterpret_cast<const uint32_t*>(g.s2.dig), (const int*)g.s2.dexp,
             (const double*)g.s2.dsum, (const double*)g.s2.cm, g.m2.off, g.m2.base, g.m2.ent,
             g.l1t_rows_pad, g.s2.part);
}
}  // namespace

// main kernel alone, fully serialized (the roofline timing in gkb_op_bench)
void k1_main_only(const GenoView& g, const double* x, cudaStream_t s) {
  if (g.ind) {
    launch_ind<0>(g, g.pl1, g.lt1, g.s1, s, false);
    return;
  }
  launch_main<0>(g, g.pl1, g.lt1, g.s1, x, g.m1, s, false);
}

void k2_main_only(const GenoView& g, cudaStream_t s) {
  if (g.single) {
    launch_adj_l1(g, s, false);
    return;
  }
  if (g.ind) {
    launch_ind<1>(g, g.pl2, g.lt2, g.s2, s, false);
    return;
  }
  launch_main<1>(g, g.pl2, g.lt2, g.s2, g.s2.cm, g.m2, s, false);
}

void k1_apply(const GenoView& g, const double* x, double* y, cudaStream_t s, bool stream_out,
              const DivIn& di) {
  if (g.p_loc == 0) {
    if (di.div) div_copy_dv(x, di.div, di.store, g.n, s, di.gate);
    return;
  }
  k1_digitize(g, x, s, di);
  if (di.div) x = di.store;  // the missing-entry terms read the stored quotient
  if (g.ind) {
    launch_ind<0>(g, g.pl1, g.lt1, g.s1, s, true);
    launch_pdl(k1_reduce, dim3((unsigned)((g.p_loc + 255) / 256)), dim3(256), 0, s, true,
               (const double*)g.s1.part, g.pl1.nkc, g.pl1.rows_pad, g.p_loc,
               (const double*)g.inv_s, y);
    return;
  }
  if (stream_out) {  // finish fused into the last CTA of each row block: y rows leave progressively
    launch_main<0>(g, g.pl1, g.lt1, g.s1, x, g.m1, s, true, y);
    return;
  }
  launch_main<0>(g, g.pl1, g.lt1, g.s1, x, g.m1, s, true);
  launch_pdl(k1_reduce, dim3((unsigned)((g.p_loc + 255) / 256)), dim3(256), 0, s, true,
             (const double*)g.s1.part, g.pl1.nkc, g.pl1.rows_pad, g.p_loc, (const double*)g.inv_s,
             y);
}

void k2_adjoint(const GenoView& g, const double* y, double* z, cudaStream_t s, const DivIn& di) {
  if (g.n == 0 || g.p_loc == 0) {
    if (di.div) div_copy_dv(y, di.div, di.store, g.p_loc, s, di.gate);
    if (g.n > 0) cudaMemsetAsync(z, 0, sizeof(double) * (size_t)g.n, s);
    return;
  }
  if (g.single) {  // K2 from layout 1
    digitize_l1t(g, y, s, di);
    launch_adj_l1(g, s, true);
    launch_k2_reduce((const double*)g.s2.part, (int)g.l1t_nkc, g.l1t_rows_pad, g.n, z, s);
    return;
  }
  k2_digitize(g, y, s, di);  // (+ the cm digits in dense-missing mode)
  if (g.ind) {
    launch_ind<1>(g, g.pl2, g.lt2, g.s2, s, true);
  } else {
    launch_main<1>(g, g.pl2, g.lt2, g.s2, g.s2.cm, g.m2, s, true);
  }
  launch_k2_reduce((const double*)g.s2.part, g.pl2.nkc, g.pl2.rows_pad, g.n, z, s);
}

// ---- tcgen05 block products ------------------------------------------------
int tc_nkc(const PMPlan& pl) { return (int)((pl.KT + kTcSpan - 1) / kTcSpan); }

size_t tc_dig_bytes(const PMPlan& pl, int kmax) {
  const int kp = kmax + (kmax & 1);
  return (size_t)tc_nkc(pl) * kTcSpan * (size_t)(8 * kp) * 128;
}

namespace {
template <int MODE>
void launch_tc(const GenoView& g, const PMPlan& pl, const uint4* lay, const TcScratch& t, int k,
               cudaStream_t s) {
  const size_t smem = tc_smem_bytes(k + (k & 1), MODE);
  allow_smem(k_pm_blk_tc<MODE>, smem);
  const int nkc = tc_nkc(pl);
  launch_pdl(k_pm_blk_tc<MODE>, dim3((unsigned)pl.grid_x, (unsigned)nkc), dim3(kThreads + 32),
             smem, s, true, lay, pl.KT, kTcSpan, k, k + (k & 1), (const uint8_t*)t.dig,
             (const uint8_t*)t.dig2, (const int*)t.dexp, (const int*)t.dexp2,
             (const double*)t.dsum, (const double*)g.mu, (const double*)g.mean, pl.rows_pad, nkc,
             t.part);
}
}  // namespace

void k1_apply_tc(const GenoView& g, const TcScratch& t, const double* X, int64_t ldx, int k,
                 double* Y, int64_t ldy, cudaStream_t s) {
  if (g.p_loc == 0 || k <= 0) return;
  const PMPlan& pl = g.pl1;
  const int nkc = tc_nkc(pl);
  const size_t dsm = (size_t)kTcSpan * 1024;
  allow_smem(k_digitize_tc<0>, dsm);
  launch_pdl(k_digitize_tc<0>, dim3((unsigned)nkc, (unsigned)(k + (k & 1))), dim3(1024), dsm, s,
             true, X, ldx, k, (const double*)nullptr, (const double*)nullptr,
             (const double*)nullptr, g.n, kTcSpan, t.dig, (uint8_t*)nullptr, t.dexp, (int*)nullptr,
             t.dsum);
  launch_tc<0>(g, pl, g.lt1, t, k, s);
  for (int v = 0; v < k; ++v)
    launch_pdl(k1_reduce, dim3((unsigned)((g.p_loc + 255) / 256)), dim3(256), 0, s, true,
               (const double*)(t.part + (size_t)v * nkc * pl.rows_pad), nkc, pl.rows_pad,
               g.p_loc, (const double*)g.inv_s, Y + (size_t)v * ldy);
}

void k2_adjoint_tc(const GenoView& g, const TcScratch& t, const double* Yin, int64_t ldy, int k,
                   double* Z, int64_t ldz, cudaStream_t s) {
  if (g.n == 0 || k <= 0) return;
  if (g.p_loc == 0) {
    for (int v = 0; v < k; ++v) cudaMemsetAsync(Z + (size_t)v * ldz, 0, sizeof(double) * g.n, s);
    return;
  }
  const PMPlan& pl = g.pl2;
  const int nkc = tc_nkc(pl);
  const size_t dsm = (size_t)kTcSpan * 2048;
  allow_smem(k_digitize_tc<1>, dsm);
  launch_pdl(k_digitize_tc<1>, dim3((unsigned)nkc, (unsigned)(k + (k & 1))), dim3(1024), dsm, s,
             true, Yin, ldy, k, (const double*)g.inv_s, (const double*)g.mu,
             (const double*)g.mean, g.p_loc, kTcSpan, t.dig, t.dig2, t.dexp, t.dexp2, t.dsum);
  launch_tc<1>(g, pl, g.lt2, t, k, s);
  for (int v = 0; v < k; ++v)
    launch_k2_reduce((const double*)(t.part + (size_t)v * nkc * pl.rows_pad), nkc, pl.rows_pad, g.n,
               Z + (size_t)v * ldz, s);
}

// ---- two vectors per pass (block products) ------------------------------
namespace {
template <int MODE>
void digitize_into(const GenoView& g, const PMPlan& pl, const double* v, const PMScratch& sc,
                   cudaStream_t s, bool pdl) {
  allow_smem(k_digitize<MODE>, pl.dig_smem);
  if (MODE == 0)
    launch_pdl(k_digitize<0>, dim3((unsigned)pl.nkc), dim3(1024), pl.dig_smem, s, pdl, v,
               (const double*)nullptr, (const double*)nullptr, (const double*)nullptr, g.n,
               pl.kt_cta, sc.dig, sc.dexp, sc.dsum, (double*)nullptr, (const double*)nullptr,
               (double*)nullptr, (const int*)nullptr, (uint4*)nullptr, (int*)nullptr);
  else
    launch_pdl(k_digitize<1>, dim3((unsigned)pl.nkc), dim3(1024), pl.dig_smem, s, pdl, v,
               (const double*)g.inv_s, (const double*)g.mu, (const double*)g.mean, g.p_loc,
               pl.kt_cta, sc.dig, sc.dexp, sc.dsum, sc.cm, (const double*)nullptr, (double*)nullptr,
               (const int*)nullptr, (uint4*)nullptr, (int*)nullptr);
}

template <int MODE>
void launch_main2(const GenoView& g, const PMPlan& pl, const uint4* lay, const PMScratch& s0,
                  const PMScratch& s1, const double* cv0, const double* cv1, const MissLists& ml,
                  cudaStream_t s) {
  const size_t smem = pm2_smem_bytes(pl.kt_cta);
  allow_smem(k_pm_main2<MODE>, smem);
  PM2Args a;
  a.dig[0] = s0.dig;
  a.dig[1] = s1.dig;
  a.dexp[0] = s0.dexp;
  a.dexp[1] = s1.dexp;
  a.dsum[0] = s0.dsum;
  a.dsum[1] = s1.dsum;
  a.cval[0] = cv0;
  a.cval[1] = cv1;
  a.part[0] = s0.part;
  a.part[1] = s1.part;
  launch_pdl(k_pm_main2<MODE>, dim3((unsigned)pl.grid_x, (unsigned)pl.nkc), dim3(kThreads), smem,
             s, true, lay, pl.KT, pl.kt_cta, a, (const double*)g.mu, (const double*)g.mean,
             ml.off, ml.base, ml.ent, pl.rows_pad, pl.C);
}
}  // namespace

void k1_apply2(const GenoView& g, const PMScratch& sb, const double* x0, const double* x1,
               double* y0, double* y1, cudaStream_t s) {
  if (g.p_loc == 0) return;
  if (g.ind) {  // dense-missing mode: two single-vector products
    k1_apply(g, x0, y0, s, false, DivIn{});
    k1_apply(g, x1, y1, s, false, DivIn{});
    return;
  }
  digitize_into<0>(g, g.pl1, x0, g.s1, s, true);
  digitize_into<0>(g, g.pl1, x1, sb, s, true);
  launch_main2<0>(g, g.pl1, g.lt1, g.s1, sb, x0, x1, g.m1, s);
  for (int v = 0; v < 2; ++v)
    launch_pdl(k1_reduce, dim3((unsigned)((g.p_loc + 255) / 256)), dim3(256), 0, s, true,
               (const double*)(v ? sb.part : g.s1.part), g.pl1.nkc, g.pl1.rows_pad, g.p_loc,
               (const double*)g.inv_s, v ? y1 : y0);
}

void k2_adjoint2(const GenoView& g, const PMScratch& sb, const double* y0, const double* y1,
                 double* z0, double* z1, cudaStream_t s) {
  if (g.n == 0) return;
  if (g.p_loc == 0) {
    cudaMemsetAsync(z0, 0, sizeof(double) * (size_t)g.n, s);
    cudaMemsetAsync(z1, 0, sizeof(double) * (size_t)g.n, s);
    return;
  }
  if (g.ind || g.single) {  // dense-missing / single-layout mode: two single-vector products
    k2_adjoint(g, y0, z0, s, DivIn{});
    k2_adjoint(g, y1, z1, s, DivIn{});
    return;
  }
  digitize_into<1>(g, g.pl2, y0, g.s2, s, true);
  digitize_into<1>(g, g.pl2, y1, sb, s, true);
  launch_main2<1>(g, g.pl2, g.lt2, g.s2, sb, g.s2.cm, sb.cm, g.m2, s);
  for (int v = 0; v < 2; ++v)
    launch_k2_reduce((const double*)(v ? sb.part : g.s2.part), g.pl2.nkc, g.pl2.rows_pad, g.n,
               v ? z1 : z0, s);
}

void marker_scan(const GenoView& g, const double* P, int64_t ldp, int K, const double* Ainv,
                 const double* w, double yyc, double a0w, double denom, const int64_t* counts,
                 double* beta, double* se, double* icpt, double* sig2, int* dep,
                 cudaStream_t s) {
  if (g.p_loc == 0) return;
  const size_t sm = sizeof(double) * (size_t)(K * K + K);
  launch_pdl(k_marker_scan, dim3((unsigned)std::min<int64_t>((g.p_loc + 255) / 256, 148 * 8)),
             dim3(256), sm, s, true, P, ldp, g.p_loc, K, Ainv, w, yyc, a0w, denom, counts,
             (const double*)g.mu, (const double*)g.inv_s, (const double*)g.mean, beta, se, icpt,
             sig2, dep);
}

}  // namespace dev
}  // namespace gkb
