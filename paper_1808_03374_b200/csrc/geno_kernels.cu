// Packed-genotype kernels for sm_100a: layout build (K8), marker counts (K7),
// missing-entry lists, K1 = reference apply (X x, per-SNP dot) and
// K2 = reference apply_adjoint (X^T y, per-sample sum).
//
// Reference semantics (/root/reference/proj):
//   .bed code table            genio.cpp:33   (00->2, 01->missing, 10->1, 11->0)
//   standardized entry          genio.cpp:124-185: (d - mu_j)/s_j, missing -> 0
//   DenseOperator apply/adjoint linop.hpp:50-58
//
// Decode ("denormal injection"): each 2-bit dosage code r
// of a 32-bit word is masked in place with one LOP3 and used as the low word
// of an fp64 operand whose high word is 0, i.e. the denormal r * 2^(2k-1074)
// for field k. One DFMA per genotype accumulates it against a coefficient
// pre-scaled by 2^(S - E - 2k) (K1) or 2^(S - E) (K2), where E is the block's
// largest coefficient exponent; products are exact-normal fp64 numbers and
// the accumulator is rescaled once with scalbn. No constant offset is added,
// so no precision is lost to cancellation; every sum is a plain fp64 sum in a
// fixed order.
//
// Missing entries are stored as r = 3 in the layouts (so the layouts retain
// the full .bed information); their 3*coef contribution is removed exactly
// by sparse corrections over sorted missing lists in the reduce kernels.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace gkb {
namespace dev {

namespace {

constexpr int kS = 1000;  // coefficient scale exponent (see header comment)
constexpr int kThreads = 256;
constexpr int kDepth = 4;  // 16-byte loads in flight per thread in the main loops
constexpr int kSubQ = 64;  // SNP quads per pair-table sub-chunk in k2_main_h (8 KB of tables)

__device__ __forceinline__ double fld(uint32_t w, int k) {
  return __hiloint2double(0, (int)(w & (3u << (2 * k))));
}

// .bed 2-bit code -> dosage code r (r_hi = ~h, r_lo = l ^ h per field).
__device__ __forceinline__ uint32_t bed_to_r(uint32_t c) {
  return ((~c) & 0xAAAAAAAAu) | ((c ^ (c >> 1)) & 0x55555555u);
}
// inverse mapping r -> .bed code
__device__ __forceinline__ uint32_t r_to_bed(uint32_t r) {
  return ((~r) & 0xAAAAAAAAu) | ((r ^ ((~r) >> 1)) & 0x55555555u);
}
__device__ __forceinline__ uint32_t missing_mask(uint32_t r) { return r & (r >> 1) & 0x55555555u; }

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
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

// ---------------------------------------------------------------- K8 / K7
__global__ void k_build_layouts(const uint8_t* __restrict__ bed, int64_t stride, int64_t rows,
                                int64_t q_base, int64_t n, int64_t W, int64_t P4,
                                uint4* __restrict__ layA, uint4* __restrict__ layB) {
  const int64_t nq = (rows + 3) / 4;
  const int64_t total = nq * W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qq = idx / W, w = idx - qq * W;
    const int64_t valid = n - 16 * w;
    const uint32_t pad_mask = valid >= 16 ? 0xFFFFFFFFu : ((1u << (2 * valid)) - 1u);
    uint32_t words[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = 4 * qq + i;
      uint32_t v = 0;
      if (row < rows) {
        const uint8_t* rec = bed + row * stride;
        const int64_t b0 = 4 * w;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (b0 + t < stride) v |= (uint32_t)rec[b0 + t] << (8 * t);
        v = bed_to_r(v) & pad_mask;
      }
      words[i] = v;
    }
    const uint4 c = make_uint4(words[0], words[1], words[2], words[3]);
    const int64_t q = q_base + qq;
    layA[q * W + w] = c;
    layB[w * P4 + q] = c;
  }
}

// one warp per SNP quad
__global__ void k_marker_counts(const uint4* __restrict__ layA, int64_t P4, int64_t W,
                                int64_t p_loc, int64_t n, int64_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < P4; q += warps) {
    int c1[4] = {0, 0, 0, 0}, c2[4] = {0, 0, 0, 0}, c3[4] = {0, 0, 0, 0};
    for (int64_t w = lane; w < W; w += 32) {
      const uint4 v = layA[q * W + w];
      const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t r = ws[i], hi = (r >> 1) & 0x55555555u, lo = r & 0x55555555u;
        c3[i] += __popc(hi & lo);
        c2[i] += __popc(hi & ~lo);
        c1[i] += __popc(~hi & lo & 0x55555555u);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      for (int o = 16; o > 0; o >>= 1) {
        c1[i] += __shfl_down_sync(0xffffffffu, c1[i], o);
        c2[i] += __shfl_down_sync(0xffffffffu, c2[i], o);
        c3[i] += __shfl_down_sync(0xffffffffu, c3[i], o);
      }
    if (lane == 0) {
      for (int i = 0; i < 4; ++i) {
        const int64_t j = 4 * q + i;
        if (j >= p_loc) break;
        counts[4 * j + 0] = n - c1[i] - c2[i] - c3[i];
        counts[4 * j + 1] = c1[i];
        counts[4 * j + 2] = c2[i];
        counts[4 * j + 3] = c3[i];
      }
    }
  }
}

// thread per word position: counts missing per sample over all local SNPs
__global__ void k_sample_missing_counts(const uint4* __restrict__ layA, int64_t P4, int64_t W,
                                        int64_t p_loc, int64_t n, int64_t* __restrict__ col_counts) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  int cnt[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) cnt[k] = 0;
  for (int64_t q = 0; q < P4; ++q) {
    const uint4 v = layA[q * W + w];
    const uint32_t m = missing_mask(v.x) | (missing_mask(v.y) << 1);
    const uint32_t m2 = missing_mask(v.z) | (missing_mask(v.w) << 1);
    if ((m | m2) == 0) continue;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      cnt[k] += ((m >> (2 * k)) & 1u) + ((m >> (2 * k + 1)) & 1u) + ((m2 >> (2 * k)) & 1u) +
                ((m2 >> (2 * k + 1)) & 1u);
  }
  (void)p_loc;  // pad SNP rows are r = 0, never missing
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (16 * w + k < n) col_counts[16 * w + k] = cnt[k];
}

// warp per SNP row: sorted sample ids of its missing entries
__global__ void k_fill_missing_rows(const uint4* __restrict__ layA, int64_t P4, int64_t W,
                                    int64_t p_loc, const int64_t* __restrict__ row_ptr,
                                    int32_t* __restrict__ row_idx) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < p_loc; j += warps) {
    const int64_t q = j >> 2;
    const int i = (int)(j & 3);
    if (row_ptr[j + 1] == row_ptr[j]) continue;
    int64_t base = row_ptr[j];
    for (int64_t w0 = 0; w0 < W; w0 += 32) {
      const int64_t w = w0 + lane;
      uint32_t m = 0;
      if (w < W) {
        const uint4 v = layA[q * W + w];
        const uint32_t r = i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
        m = missing_mask(r);
      }
      const int c = __popc(m);
      int incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int64_t pos = base + incl - c;
      while (m) {
        const int b = __ffs(m) - 1;
        row_idx[pos++] = (int32_t)(16 * w + (b >> 1));
        m &= m - 1;
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// thread per word position: sorted local SNP ids per sample (ascending j)
__global__ void k_fill_missing_cols(const uint4* __restrict__ layA, int64_t P4, int64_t W,
                                    int64_t p_loc, int64_t n, const int64_t* __restrict__ col_ptr,
                                    int32_t* __restrict__ col_idx) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  int64_t cur[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) cur[k] = (16 * w + k < n) ? col_ptr[16 * w + k] : 0;
  for (int64_t q = 0; q < P4; ++q) {
    const uint4 v = layA[q * W + w];
    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
    if ((missing_mask(v.x) | missing_mask(v.y) | missing_mask(v.z) | missing_mask(v.w)) == 0)
      continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t m = missing_mask(ws[i]);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if ((m >> (2 * k)) & 1u) col_idx[cur[k]++] = (int32_t)(4 * q + i);
    }
  }
  (void)p_loc;
}

__global__ void k_layout_to_bed(const uint4* __restrict__ layA, int64_t P4, int64_t W, int64_t n,
                                int64_t row0, int64_t nrows, uint8_t* __restrict__ out) {
  const int64_t stride = (n + 3) / 4;
  const int64_t total = nrows * W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = idx / W, w = idx - rr * W;
    const int64_t j = row0 + rr;
    const uint4 v = layA[(j >> 2) * W + w];
    const int i = (int)(j & 3);
    const uint32_t r = i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
    uint32_t c = r_to_bed(r);
    const int64_t valid = n - 16 * w;
    if (valid < 16) c &= (1u << (2 * valid)) - 1u;  // pads 00 (genio.cpp:100)
    uint8_t* rec = out + rr * stride;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * w + t < stride) rec[4 * w + t] = (uint8_t)(c >> (8 * t));
  }
}

// ---------------------------------------------------------------- K1 apply
// One 16-byte chunk: 4 SNP words x 16 samples against the 16 (scaled) sample
// coefficients of that word position.
__device__ __forceinline__ void k1_word(const uint4 c, const double2* __restrict__ cf, double& a0,
                                        double& a1, double& a2, double& a3) {
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const double2 xx = cf[kk];
    a0 = fma(fld(c.x, 2 * kk), xx.x, a0);
    a1 = fma(fld(c.y, 2 * kk), xx.x, a1);
    a2 = fma(fld(c.z, 2 * kk), xx.x, a2);
    a3 = fma(fld(c.w, 2 * kk), xx.x, a3);
    a0 = fma(fld(c.x, 2 * kk + 1), xx.y, a0);
    a1 = fma(fld(c.y, 2 * kk + 1), xx.y, a1);
    a2 = fma(fld(c.z, 2 * kk + 1), xx.y, a2);
    a3 = fma(fld(c.w, 2 * kk + 1), xx.y, a3);
  }
}

// One 16-byte chunk of layout A: 4 SNP words x the lane's 16 samples.
__device__ __forceinline__ void k2_quad(const uint4 c, const double2 ca, const double2 cb,
                                        double (&acc)[16]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = fma(fld(c.x, k), ca.x, acc[k]);
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = fma(fld(c.y, k), ca.y, acc[k]);
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = fma(fld(c.z, k), cb.x, acc[k]);
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = fma(fld(c.w, k), cb.y, acc[k]);
}
// grid (ceil(P4/32), ntiles). Lane = SNP quad q (4 SNPs), loops over the
// tile's word positions; lanes read 32 consecutive 16-byte chunks (512 B).
__global__ void __launch_bounds__(kThreads) k1_main(const uint4* __restrict__ layB, int64_t P4,
                                                    int64_t W, const double* __restrict__ x,
                                                    int64_t n, int tileW,
                                                    double* __restrict__ ypart,
                                                    double* __restrict__ xsum) {
  extern __shared__ double2 xp2[];  // tileW * 8 double2: scaled coefficients
  __shared__ double red[33];
  __shared__ int redi[33];
  double* xp = reinterpret_cast<double*>(xp2);
  const int tile = blockIdx.y;
  const int64_t w0 = (int64_t)tile * tileW;
  const int64_t w1 = min(W, w0 + tileW);
  const int nw = (int)(w1 - w0);
  const int ns = nw * 16;

  int emax = -1100;
  double part = 0.0;
  for (int t = threadIdx.x; t < ns; t += kThreads) {
    const int64_t sidx = 16 * w0 + t;
    const double xv = sidx < n ? x[sidx] : 0.0;
    emax = max(emax, exp_of(xv));
    part += xv;
    xp[t] = xv;
  }
  const int E = block_max_int(emax, redi);
  const double tsum = block_sum(part, red);
  for (int t = threadIdx.x; t < ns; t += kThreads) xp[t] = scalbn(xp[t], kS - E - 2 * (t & 15));
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) xsum[tile] = tsum;

  // Lane = SNP quad (32 consecutive quads per CTA, 512-B coalesced rows of
  // layout B); warp w takes the w-th eighth of the tile's word positions, and
  // the 8 warp partials are added in warp order through shared memory.
  __shared__ double wsum[8][4][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * 32 + lane;
  const int sub = (nw + 7) / 8;
  const int wa = min(nw, warp * sub), we = min(nw, wa + sub);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (q < P4 && wa < we) {
    const uint4* src = layB + w0 * P4 + q;
    const uint4 Z = make_uint4(0, 0, 0, 0);
    // four 16-byte loads in flight per thread; each slot is refilled right
    // after it is consumed (no dynamic indexing, no early exits)
    uint4 c0 = ld_stream(src + (int64_t)wa * P4);
    uint4 c1 = wa + 1 < we ? ld_stream(src + (int64_t)(wa + 1) * P4) : Z;
    uint4 c2 = wa + 2 < we ? ld_stream(src + (int64_t)(wa + 2) * P4) : Z;
    uint4 c3 = wa + 3 < we ? ld_stream(src + (int64_t)(wa + 3) * P4) : Z;
    int w = wa;
    for (; w + 4 <= we; w += 4) {
      k1_word(c0, xp2 + 8 * w, a0, a1, a2, a3);
      c0 = w + 4 < we ? ld_stream(src + (int64_t)(w + 4) * P4) : Z;
      k1_word(c1, xp2 + 8 * (w + 1), a0, a1, a2, a3);
      c1 = w + 5 < we ? ld_stream(src + (int64_t)(w + 5) * P4) : Z;
      k1_word(c2, xp2 + 8 * (w + 2), a0, a1, a2, a3);
      c2 = w + 6 < we ? ld_stream(src + (int64_t)(w + 6) * P4) : Z;
      k1_word(c3, xp2 + 8 * (w + 3), a0, a1, a2, a3);
      c3 = w + 7 < we ? ld_stream(src + (int64_t)(w + 7) * P4) : Z;
    }
    if (w < we) k1_word(c0, xp2 + 8 * w, a0, a1, a2, a3);
    if (w + 1 < we) k1_word(c1, xp2 + 8 * (w + 1), a0, a1, a2, a3);
    if (w + 2 < we) k1_word(c2, xp2 + 8 * (w + 2), a0, a1, a2, a3);
  }
  wsum[warp][0][lane] = a0;
  wsum[warp][1][lane] = a1;
  wsum[warp][2][lane] = a2;
  wsum[warp][3][lane] = a3;
  __syncthreads();
  if (threadIdx.x < 128) {
    const int i = threadIdx.x >> 5;  // SNP within the quad
    const int64_t qq = (int64_t)blockIdx.x * 32 + lane;
    if (qq < P4) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += wsum[w][i][lane];
      ypart[(int64_t)tile * 4 * P4 + 4 * qq + i] = scalbn(t, 1074 - kS + E);
    }
  }
}

// y_j = inv_s_j * (sum_t ypart - mu_j X_tot - (3 - mu_j) S_miss_j)
__global__ void k1_reduce(const double* __restrict__ ypart, const double* __restrict__ xsum,
                          int ntiles, int64_t P4, int64_t p_loc, const double* __restrict__ x,
                          const double* __restrict__ mu, const double* __restrict__ inv_s,
                          const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ row_idx,
                          double* __restrict__ y) {
  // One warp per SNP: lanes stride over the sample tiles and over the SNP's
  // sorted missing list; fixed shuffle tree -> deterministic.
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double xt = 0.0;
  for (int t = lane; t < ntiles; t += 32) xt += xsum[t];
  for (int o = 16; o > 0; o >>= 1) xt += __shfl_xor_sync(0xffffffffu, xt, o);
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < p_loc; j += nwarps) {
    double acc = 0.0, sm = 0.0;
    for (int t = lane; t < ntiles; t += 32) acc += ypart[(int64_t)t * 4 * P4 + j];
    if (row_ptr) {
      const int64_t e0 = row_ptr[j], e1 = row_ptr[j + 1];
#pragma unroll 8
      for (int64_t e = e0 + lane; e < e1; e += 32) sm += x[row_idx[e]];
    }
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_down_sync(0xffffffffu, acc, o);
      sm += __shfl_down_sync(0xffffffffu, sm, o);
    }
    if (lane == 0) {
      const double m = mu[j];
      y[j] = inv_s[j] * (acc - m * xt - (3.0 - m) * sm);
    }
  }
}

// ---------------------------------------------------------------- K2 adjoint
// grid (ceil(W/32), nchunks). Lane = word position w (16 samples, 16
// accumulators); loops over the chunk's SNP quads; lanes read 32 consecutive
// 16-byte chunks of one quad row (512 B).
__global__ void __launch_bounds__(kThreads, 4) k2_main(const uint4* __restrict__ layA, int64_t P4,
                                                    int64_t W, const double* __restrict__ y,
                                                    const double* __restrict__ mu,
                                                    const double* __restrict__ inv_s,
                                                    int64_t p_loc, int qc,
                                                    double* __restrict__ zpart,
                                                    double* __restrict__ kpart,
                                                    double* __restrict__ cmiss) {
  extern __shared__ double2 cs2[];  // 2*qc double2 = 4*qc scaled coefficients
  __shared__ double red[33];
  __shared__ int redi[33];
  double* cs = reinterpret_cast<double*>(cs2);
  const int chunk = blockIdx.y;
  const int64_t q0 = (int64_t)chunk * qc;
  const int64_t q1 = min(P4, q0 + qc);
  const int nq = (int)(q1 - q0);

  int emax = -1100;
  double kp = 0.0;
  for (int t = threadIdx.x; t < 4 * nq; t += kThreads) {
    const int64_t j = 4 * q0 + t;
    const double c = j < p_loc ? inv_s[j] * y[j] : 0.0;
    emax = max(emax, exp_of(c));
    if (j < p_loc) {
      kp += c * mu[j];
      if (cmiss && blockIdx.x == 0) cmiss[j] = c * (3.0 - mu[j]);  // missing-entry correction
    }
    cs[t] = c;
  }
  const int E = block_max_int(emax, redi);
  const double ksum = block_sum(kp, red);
  for (int t = threadIdx.x; t < 4 * nq; t += kThreads) cs[t] = scalbn(cs[t], kS - E);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) kpart[chunk] = ksum;

  // Lane = word position (32 consecutive words, 512-B coalesced rows of
  // layout A); warp w takes the w-th eighth of the chunk's SNP quads; the 8
  // warp partials are added in warp order through shared memory.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = (int64_t)blockIdx.x * 32 + lane;
  const int sub = (nq + 7) / 8;
  const int qa = min(nq, warp * sub), qe = min(nq, qa + sub);
  double acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  if (w < W && qa < qe) {
    const uint4* src = layA + q0 * W + w;
    const uint4 Z = make_uint4(0, 0, 0, 0);
    uint4 c0 = ld_stream(src + (int64_t)qa * W);
    uint4 c1 = qa + 1 < qe ? ld_stream(src + (int64_t)(qa + 1) * W) : Z;
    uint4 c2 = qa + 2 < qe ? ld_stream(src + (int64_t)(qa + 2) * W) : Z;
    uint4 c3 = qa + 3 < qe ? ld_stream(src + (int64_t)(qa + 3) * W) : Z;
    int qq = qa;
    for (; qq + 4 <= qe; qq += 4) {
      k2_quad(c0, cs2[2 * qq], cs2[2 * qq + 1], acc);
      c0 = qq + 4 < qe ? ld_stream(src + (int64_t)(qq + 4) * W) : Z;
      k2_quad(c1, cs2[2 * qq + 2], cs2[2 * qq + 3], acc);
      c1 = qq + 5 < qe ? ld_stream(src + (int64_t)(qq + 5) * W) : Z;
      k2_quad(c2, cs2[2 * qq + 4], cs2[2 * qq + 5], acc);
      c2 = qq + 6 < qe ? ld_stream(src + (int64_t)(qq + 6) * W) : Z;
      k2_quad(c3, cs2[2 * qq + 6], cs2[2 * qq + 7], acc);
      c3 = qq + 7 < qe ? ld_stream(src + (int64_t)(qq + 7) * W) : Z;
    }
    if (qq < qe) k2_quad(c0, cs2[2 * qq], cs2[2 * qq + 1], acc);
    if (qq + 1 < qe) k2_quad(c1, cs2[2 * qq + 2], cs2[2 * qq + 3], acc);
    if (qq + 2 < qe) k2_quad(c2, cs2[2 * qq + 4], cs2[2 * qq + 5], acc);
  }
  // cross-warp combine in two halves of 8 fields (16 KB of the coefficient
  // region, which is sized >= 2048 doubles)
  double* part = cs;
  const int k_out = threadIdx.x >> 5;  // field within the half, 0..7
  const int64_t w_out = (int64_t)blockIdx.x * 32 + lane;
  double* out = zpart + (int64_t)chunk * 16 * W;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) part[(warp * 8 + k) * 32 + lane] = acc[8 * h + k];
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) t += part[(ww * 8 + k_out) * 32 + lane];
    const int field = 8 * h + k_out;
    if (w_out < W) out[16 * w_out + field] = scalbn(t, 1074 - kS + E - 2 * field);
  }
}

// ---------------------------------------------------------------- K2 hybrid
// Same contract as k2_main, but the work of every SNP quad is split across
// two pipes: SNPs (4q, 4q+1) go through a 16-entry fp64 pair table in shared
// memory -- T_q[r_a | r_b << 2] = v_a(r_a) + v_b(r_b), v_j(r) = c_j (r - mu_j)
// for r <= 2 and 0 for a missing entry -- so each lookup (one PRMT address
// op, one LDS.64, one DADD) covers two genotypes on the LSU pipe; SNPs
// (4q+2, 4q+3) go through the denormal-injection DFMA path on the FP64 pipe.
// Table-path SNPs need no missing correction (cmiss = 0) and no mu term.
// Lane = half a word (8 samples): lanes 2i, 2i+1 share word w0 + i.
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));  // tables are read-only after setup
  return v;
}

__global__ void __launch_bounds__(kThreads) k2_main_h(const uint4* __restrict__ layA, int64_t P4,
                                                      int64_t W, const double* __restrict__ y,
                                                      const double* __restrict__ mu,
                                                      const double* __restrict__ inv_s,
                                                      int64_t p_loc, int qc,
                                                      double* __restrict__ zpart,
                                                      double* __restrict__ kpart,
                                                      double* __restrict__ cmiss) {
  extern __shared__ __align__(16) double sm_raw[];
  // tables start on a 256-byte boundary: table qq is at byte (qq>>1)*256 + (qq&1)*128
  const uint32_t raw_addr = (uint32_t)__cvta_generic_to_shared(sm_raw);
  double* sm2 = sm_raw + (((raw_addr + 255u) & ~255u) - raw_addr) / 8;
  double* tabs = sm2;                                            // kSubQ * 16 (128 B per quad)
  double2* csd = reinterpret_cast<double2*>(sm2 + 16 * kSubQ);   // qc scaled (c_{4q+2}, c_{4q+3})
  __shared__ double red[33];
  __shared__ int redi[33];
  const int chunk = blockIdx.y;
  const int64_t q0 = (int64_t)chunk * qc;
  const int64_t q1 = min(P4, q0 + qc);
  const int nq = (int)(q1 - q0);

  // DFMA-path coefficients (SNPs 4q+2, 4q+3) of the whole chunk: exponent,
  // mu term and missing corrections
  int emax = -1100;
  double kp = 0.0;
  for (int t = threadIdx.x; t < 2 * nq; t += kThreads) {
    const int64_t j = 4 * (q0 + (t >> 1)) + 2 + (t & 1);
    const double c = j < p_loc ? inv_s[j] * y[j] : 0.0;
    emax = max(emax, exp_of(c));
    if (j < p_loc) kp += c * mu[j];
    reinterpret_cast<double*>(csd)[t] = c;
  }
  if (cmiss && blockIdx.x == 0)
    for (int t = threadIdx.x; t < 4 * nq; t += kThreads) {
      const int64_t j = 4 * q0 + t;
      if (j < p_loc) cmiss[j] = (t & 2) ? inv_s[j] * y[j] * (3.0 - mu[j]) : 0.0;
    }
  const int E = block_max_int(emax, redi);
  const double ksum = block_sum(kp, red);
  for (int t = threadIdx.x; t < 2 * nq; t += kThreads)
    reinterpret_cast<double*>(csd)[t] = scalbn(reinterpret_cast<double*>(csd)[t], kS - E);
  if (blockIdx.x == 0 && threadIdx.x == 0) kpart[chunk] = ksum;

  // Warps split the CTA's 128 word positions (16 per warp, two lanes per
  // word); every warp walks all quads of the chunk, kSubQ at a time, against
  // pair tables shared by the whole CTA.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane & 1;
  const int64_t w = (int64_t)blockIdx.x * 128 + warp * 16 + (lane >> 1);
  const bool active = w < W;
  const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tabs);
  const uint32_t sel_h = half ? 0x00007632u : 0x00005410u;  // bytes (2h, 2h+1) of te | to
  const int sh = 16 * half;
  const uint4* src = layA + q0 * W + (active ? w : 0);
  double at[8], ad[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    at[k] = 0.0;
    ad[k] = 0.0;
  }
  for (int s0 = 0; s0 < nq; s0 += kSubQ) {
    const int s1 = min(nq, s0 + kSubQ);
    __syncthreads();  // previous sub-chunk's tables fully consumed (and csd visible)
    // pair tables for SNPs (4q, 4q+1) of quads [s0, s1)
    for (int e = threadIdx.x; e < 16 * (s1 - s0); e += kThreads) {
      const int qq = e >> 4, n = e & 15, ra = n & 3, rb = n >> 2;
      const int64_t ja = 4 * (q0 + s0 + qq), jb = ja + 1;
      double va = 0.0, vb = 0.0;
      if (ra != 3 && ja < p_loc) va = inv_s[ja] * y[ja] * ((double)ra - mu[ja]);
      if (rb != 3 && jb < p_loc) vb = inv_s[jb] * y[jb] * ((double)rb - mu[jb]);
      tabs[e] = va + vb;
    }
    __syncthreads();
    if (!active) continue;
    const uint4 Z = make_uint4(0, 0, 0, 0);
    uint4 n0 = ld_stream(src + (int64_t)s0 * W);
    uint4 n1 = s0 + 1 < s1 ? ld_stream(src + (int64_t)(s0 + 1) * W) : Z;
    uint4 n2 = s0 + 2 < s1 ? ld_stream(src + (int64_t)(s0 + 2) * W) : Z;
    for (int qq = s0; qq < s1; ++qq) {
      const uint4 c = n0;
      n0 = n1;
      n1 = n2;
      n2 = qq + 3 < s1 ? ld_stream(src + (int64_t)(qq + 3) * W) : Z;
      // ---- table path: nibble (r_x | r_y << 2) per sample
      const uint32_t te = (c.x & 0x33333333u) | ((c.y << 2) & 0xCCCCCCCCu);  // fields 0,2,..,14
      const uint32_t to = ((c.x >> 2) & 0x33333333u) | (c.y & 0xCCCCCCCCu);  // fields 1,3,..,15
      // this lane's 8 fields: nibbles n0..n3 = fields 8h+{0,2,4,6}, n4..n7 = 8h+{1,3,5,7}
      const uint32_t tt = __byte_perm(te, to, sel_h);
      const uint32_t par = (qq & 1) ? 0x80808080u : 0u;
      const uint32_t u0 = ((tt << 3) & 0x78787878u) | par;  // n0,n2,n4,n6 -> fields 0,4,1,5
      const uint32_t u1 = ((tt >> 1) & 0x78787878u) | par;  // n1,n3,n5,n7 -> fields 2,6,3,7
      const uint32_t base = tab_addr + (uint32_t)((qq - s0) >> 1) * 256u;
      // address = table base (bytes 1..3, byte 0 == 0) with byte 0 = nibble*8 | parity*128
      at[0] += lds_f64(__byte_perm(u0, base, 0x7650u));
      at[4] += lds_f64(__byte_perm(u0, base, 0x7651u));
      at[1] += lds_f64(__byte_perm(u0, base, 0x7652u));
      at[5] += lds_f64(__byte_perm(u0, base, 0x7653u));
      at[2] += lds_f64(__byte_perm(u1, base, 0x7650u));
      at[6] += lds_f64(__byte_perm(u1, base, 0x7651u));
      at[3] += lds_f64(__byte_perm(u1, base, 0x7652u));
      at[7] += lds_f64(__byte_perm(u1, base, 0x7653u));
      // ---- DFMA path for SNPs 4q+2, 4q+3 on this lane's 8 fields
      const double2 cc = csd[qq];
      const uint32_t zz = c.z >> sh, ww = c.w >> sh;
#pragma unroll
      for (int k = 0; k < 8; ++k) ad[k] = fma(fld(zz, k), cc.x, ad[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) ad[k] = fma(fld(ww, k), cc.y, ad[k]);
    }
  }
  // lane's field f (0..7) = sample 16w + 8h + f: at[f] plain, ad[f] scaled by
  // 2^(2f + kS - E - 1074)
  if (active) {
    double2* out = reinterpret_cast<double2*>(zpart + (int64_t)chunk * 16 * W + 16 * w + 8 * half);
#pragma unroll
    for (int f = 0; f < 8; f += 2)
      out[f / 2] = make_double2(at[f] + scalbn(ad[f], 1074 - kS + E - 2 * f),
                                at[f + 1] + scalbn(ad[f + 1], 1074 - kS + E - 2 * (f + 1)));
  }
}

// z_s = sum_c zpart - sum_c kpart - sum_{j in miss(s)} cmiss_j,
// cmiss_j = inv_s_j y_j (3 - mu_j) written by k2_main.
// Block = 8 warps x 32 consecutive samples: warp w sums chunks c = w (mod 8)
// with lanes on consecutive samples (coalesced), then the 8 partials are
// added in warp order; each warp walks 4 samples' missing lists with lanes
// striding the entries. Fixed trees -> deterministic.
__global__ void __launch_bounds__(1024) k2_reduce(const double* __restrict__ zpart,
                                                  const double* __restrict__ kpart, int nchunks,
                                                  int64_t W, int64_t n,
                                                  const double* __restrict__ cmiss,
                                                  const int64_t* __restrict__ col_ptr,
                                                  const int32_t* __restrict__ col_idx,
                                                  double* __restrict__ z) {
  // Block = 32 warps x 32 consecutive samples. Warp w sums chunks c = w (mod
  // 32) with lanes on consecutive samples (coalesced), and walks sample
  // s0 + w's missing list with lanes striding the entries. Partials are added
  // in warp order -> deterministic.
  __shared__ double part[32][33];
  __shared__ double corr[32];
  __shared__ double kt_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * 32;
  const int64_t s = s0 + lane;
  double acc = 0.0;
  if (s < n)
#pragma unroll 4
    for (int c = warp; c < nchunks; c += 32) acc += zpart[(int64_t)c * 16 * W + s];
  part[warp][lane] = acc;
  {
    const int64_t ss = s0 + warp;
    double cs = 0.0;
    if (col_ptr && ss < n) {
      const int64_t e0 = col_ptr[ss], e1 = col_ptr[ss + 1];
#pragma unroll 8
      for (int64_t e = e0 + lane; e < e1; e += 32) cs += cmiss[col_idx[e]];
    }
    for (int o = 16; o > 0; o >>= 1) cs += __shfl_down_sync(0xffffffffu, cs, o);
    if (lane == 0) corr[warp] = cs;
  }
  if (warp == 1) {
    double kt = 0.0;
    for (int c = lane; c < nchunks; c += 32) kt += kpart[c];
    for (int o = 16; o > 0; o >>= 1) kt += __shfl_down_sync(0xffffffffu, kt, o);
    if (lane == 0) kt_s = kt;
  }
  __syncthreads();
  if (warp == 0 && s < n) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += part[w][lane];
    z[s] = t - kt_s - corr[lane];
  }
}

int grid_for(int64_t work, int threads, int cap = 148 * 16) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

void build_layouts(const uint8_t* bed, int64_t stride_bytes, int64_t rows_in_block, int64_t q_base,
                   int64_t n, int64_t W, int64_t P4, uint4* layA, uint4* layB, cudaStream_t s) {
  const int64_t work = ((rows_in_block + 3) / 4) * W;
  if (work == 0) return;
  k_build_layouts<<<grid_for(work, 256), 256, 0, s>>>(bed, stride_bytes, rows_in_block, q_base, n,
                                                       W, P4, layA, layB);
}

void marker_counts(const uint4* layA, int64_t P4, int64_t W, int64_t p_loc, int64_t n,
                   int64_t* counts, cudaStream_t s) {
  if (P4 == 0) return;
  k_marker_counts<<<grid_for(P4 * 32, 256), 256, 0, s>>>(layA, P4, W, p_loc, n, counts);
}

void sample_missing_counts(const uint4* layA, int64_t P4, int64_t W, int64_t p_loc, int64_t n,
                           int64_t* col_counts, cudaStream_t s) {
  if (W == 0) return;
  k_sample_missing_counts<<<(unsigned)((W + 127) / 128), 128, 0, s>>>(layA, P4, W, p_loc, n,
                                                                      col_counts);
}

void fill_missing_rows(const uint4* layA, int64_t P4, int64_t W, int64_t p_loc,
                       const int64_t* row_ptr, int32_t* row_idx, cudaStream_t s) {
  if (p_loc == 0) return;
  k_fill_missing_rows<<<grid_for(p_loc * 32, 256), 256, 0, s>>>(layA, P4, W, p_loc, row_ptr,
                                                                 row_idx);
}

void fill_missing_cols(const uint4* layA, int64_t P4, int64_t W, int64_t p_loc, int64_t n,
                       const int64_t* col_ptr, int32_t* col_idx, cudaStream_t s) {
  if (W == 0) return;
  k_fill_missing_cols<<<(unsigned)((W + 127) / 128), 128, 0, s>>>(layA, P4, W, p_loc, n, col_ptr,
                                                                  col_idx);
}

void layout_to_bed(const uint4* layA, int64_t P4, int64_t W, int64_t n, int64_t row0,
                   int64_t nrows, uint8_t* out, cudaStream_t s) {
  const int64_t work = nrows * W;
  if (work == 0) return;
  k_layout_to_bed<<<grid_for(work, 256), 256, 0, s>>>(layA, P4, W, n, row0, nrows, out);
}

K1Plan k1_plan(int64_t W, int64_t P4) {
  K1Plan pl;
  // CTA = 32 SNP quads x a sample tile of 256 words (4096 samples; 32 KB of
  // coefficients), each warp 32 words. Partial traffic: 8 B per SNP per tile
  // (1/128 of the 1 KB of packed bytes per SNP and tile).
  pl.tileW = (int)(W < 256 ? (W > 0 ? W : 1) : 256);
  pl.ntiles = (int)((W + pl.tileW - 1) / pl.tileW);
  if (pl.ntiles < 1) pl.ntiles = 1;
  pl.grid_x = (P4 + 31) / 32;
  if (pl.grid_x < 1) pl.grid_x = 1;
  pl.smem = (size_t)pl.tileW * 16 * sizeof(double);
  return pl;
}

K2Plan k2_plan(int64_t W, int64_t P4) {
  K2Plan pl;
  // GKB_K2=hybrid selects the pair-table + DFMA split (k2_main_h); measured
  // slower than the DFMA-only kernel so far, so off by default.
  const char* env = getenv("GKB_K2");
  pl.hybrid = env && env[0] == 'h';
  if (pl.hybrid) {
    // CTA = 128 word positions (2048 samples; 8 warps x 16 words, two lanes
    // per word) x a chunk of up to 512 SNP quads walked in sub-chunks of
    // kSubQ quads (8 KB of pair tables). The chunk shrinks (down to kSubQ)
    // until there are >= 4 CTAs per SM; partial traffic is 8 B per sample per
    // chunk (1/64 of the packed bytes at 512 quads).
    pl.grid_x = (W + 127) / 128;
    if (pl.grid_x < 1) pl.grid_x = 1;
    int64_t want = (148 * 4 + pl.grid_x - 1) / pl.grid_x;
    int64_t qc = (P4 + want - 1) / (want > 0 ? want : 1);
    qc = ((qc + kSubQ - 1) / kSubQ) * kSubQ;
    if (qc > 512) qc = 512;
    if (qc < kSubQ) qc = kSubQ;
    pl.qc = (int)qc;
    pl.nchunks = (int)((P4 + qc - 1) / qc);
    if (pl.nchunks < 1) pl.nchunks = 1;
    pl.smem = (size_t)(16 * kSubQ + 2 * qc) * sizeof(double) + 256;
    return pl;
  }
  // CTA = 32 word positions (512 samples) x a chunk of up to 512 SNP quads
  // (2048 SNPs), each warp 64 quads. Partial traffic: 8 B per sample per
  // chunk (1/64 of the 512 packed bytes per sample and chunk).
  pl.grid_x = (W + 31) / 32;
  if (pl.grid_x < 1) pl.grid_x = 1;
  int64_t qc = 512;
  const int64_t p4r = ((P4 + 7) / 8) * 8;
  if (qc > p4r) qc = p4r > 0 ? p4r : 8;
  pl.qc = (int)qc;
  pl.nchunks = (int)((P4 + qc - 1) / qc);
  if (pl.nchunks < 1) pl.nchunks = 1;
  pl.smem = (size_t)(qc * 4 > 2048 ? qc * 4 : 2048) * sizeof(double);
  return pl;
}

void k1_main_only(const GenoView& g, const K1Plan& pl, const double* x, double* ypart, double* xsum,
                  cudaStream_t s) {
  dim3 grid((unsigned)pl.grid_x, (unsigned)pl.ntiles);
  k1_main<<<grid, kThreads, pl.smem, s>>>(g.layB, g.P4, g.W, x, g.n, pl.tileW, ypart, xsum);
}

void k1_apply(const GenoView& g, const K1Plan& pl, const double* x, double* ypart, double* xsum,
              double* y, cudaStream_t s) {
  if (g.p_loc == 0) return;
  k1_main_only(g, pl, x, ypart, xsum, s);
  k1_reduce<<<grid_for(g.p_loc * 32, 256), 256, 0, s>>>(
      ypart, xsum, pl.ntiles, g.P4, g.p_loc, x, g.mu, g.inv_s,
      g.nmissing ? g.miss_row_ptr : nullptr, g.miss_row_idx, y);
}

void k2_main_only(const GenoView& g, const K2Plan& pl, const double* y, double* zpart,
                  double* kpart, cudaStream_t s) {
  dim3 grid((unsigned)pl.grid_x, (unsigned)pl.nchunks);
  if (pl.hybrid)
    k2_main_h<<<grid, kThreads, pl.smem, s>>>(g.layA, g.P4, g.W, y, g.mu, g.inv_s, g.p_loc, pl.qc,
                                              zpart, kpart, g.nmissing ? g.cmiss : nullptr);
  else
    k2_main<<<grid, kThreads, pl.smem, s>>>(g.layA, g.P4, g.W, y, g.mu, g.inv_s, g.p_loc, pl.qc,
                                            zpart, kpart, g.nmissing ? g.cmiss : nullptr);
}

void k2_adjoint(const GenoView& g, const K2Plan& pl, const double* y, double* zpart, double* kpart,
                double* z, cudaStream_t s) {
  if (g.n == 0) return;
  if (g.p_loc == 0) {
    cudaMemsetAsync(z, 0, sizeof(double) * (size_t)g.n, s);
    return;
  }
  k2_main_only(g, pl, y, zpart, kpart, s);
  k2_reduce<<<(unsigned)((g.n + 31) / 32), 1024, 0, s>>>(
      zpart, kpart, pl.nchunks, g.W, g.n, g.cmiss, g.nmissing ? g.miss_col_ptr : nullptr,
      g.miss_col_idx, z);
}

}  // namespace dev
}  // namespace gkb
