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

#include "kernels.hpp"

namespace gkb {
namespace dev {

namespace {

constexpr int kS = 1000;  // coefficient scale exponent (see header comment)
constexpr int kThreads = 256;

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
// grid (ceil(P4/256), ntiles). Thread = SNP quad q (4 SNPs), loops over the
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

  const int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (q >= P4) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const uint4* src = layB + w0 * P4 + q;
  uint4 cn = ld_stream(src);
  for (int w = 0; w < nw; ++w) {
    const uint4 c = cn;
    if (w + 1 < nw) cn = ld_stream(src + (int64_t)(w + 1) * P4);
    const double2* cf = xp2 + 8 * w;
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
  const int un = 1074 - kS + E;
  double* out = ypart + (int64_t)tile * 4 * P4 + 4 * q;
  out[0] = scalbn(a0, un);
  out[1] = scalbn(a1, un);
  out[2] = scalbn(a2, un);
  out[3] = scalbn(a3, un);
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
    if (row_ptr)
      for (int64_t e = row_ptr[j] + lane; e < row_ptr[j + 1]; e += 32) sm += x[row_idx[e]];
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
// grid (ceil(W/256), nchunks). Thread = word position w (16 samples, 16
// accumulators); loops over the chunk's SNP quads; lanes read 32 consecutive
// 16-byte chunks of one quad row (512 B).
__global__ void __launch_bounds__(kThreads) k2_main(const uint4* __restrict__ layA, int64_t P4,
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

  const int64_t w = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (w >= W) return;
  double acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  const uint4* src = layA + q0 * W + w;
  uint4 cn = ld_stream(src);
  for (int qq = 0; qq < nq; ++qq) {
    const uint4 c = cn;
    if (qq + 1 < nq) cn = ld_stream(src + (int64_t)(qq + 1) * W);
    const double2 ca = cs2[2 * qq], cb = cs2[2 * qq + 1];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      acc[k] = fma(fld(c.x, k), ca.x, acc[k]);
      acc[k] = fma(fld(c.y, k), ca.y, acc[k]);
      acc[k] = fma(fld(c.z, k), cb.x, acc[k]);
      acc[k] = fma(fld(c.w, k), cb.y, acc[k]);
    }
  }
  double* out = zpart + (int64_t)chunk * 16 * W + 16 * w;
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const double2 v = make_double2(scalbn(acc[k], 1074 - kS + E - 2 * k),
                                   scalbn(acc[k + 1], 1074 - kS + E - 2 * (k + 1)));
    reinterpret_cast<double2*>(out)[k / 2] = v;
  }
}

// z_s = sum_c zpart - sum_c kpart - sum_{j in miss(s)} cmiss_j,
// cmiss_j = inv_s_j y_j (3 - mu_j) written by k2_main.
// Block = 8 warps x 32 consecutive samples: warp w sums chunks c = w (mod 8)
// with lanes on consecutive samples (coalesced), then the 8 partials are
// added in warp order; each warp walks 4 samples' missing lists with lanes
// striding the entries. Fixed trees -> deterministic.
__global__ void __launch_bounds__(256) k2_reduce(const double* __restrict__ zpart,
                                                 const double* __restrict__ kpart, int nchunks,
                                                 int64_t W, int64_t n,
                                                 const double* __restrict__ cmiss,
                                                 const int64_t* __restrict__ col_ptr,
                                                 const int32_t* __restrict__ col_idx,
                                                 double* __restrict__ z) {
  __shared__ double part[8][32];
  __shared__ double corr[32];
  __shared__ double kt_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * 32;
  const int64_t s = s0 + lane;
  double acc = 0.0;
  if (s < n)
    for (int c = warp; c < nchunks; c += 8) acc += zpart[(int64_t)c * 16 * W + s];
  part[warp][lane] = acc;
  for (int t = 0; t < 4; ++t) {
    const int li = warp * 4 + t;
    const int64_t ss = s0 + li;
    double cs = 0.0;
    if (col_ptr && ss < n)
      for (int64_t e = col_ptr[ss] + lane; e < col_ptr[ss + 1]; e += 32) cs += cmiss[col_idx[e]];
    for (int o = 16; o > 0; o >>= 1) cs += __shfl_down_sync(0xffffffffu, cs, o);
    if (lane == 0) corr[li] = cs;
  }
  if (threadIdx.x == 0) {
    double kt = 0.0;
    for (int c = 0; c < nchunks; ++c) kt += kpart[c];
    kt_s = kt;
  }
  __syncthreads();
  if (warp == 0 && s < n) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
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
  // A sample tile of 128 words (2048 samples): 16 KB of coefficients per CTA,
  // partial traffic 8 B per SNP per tile (1/64 of the 512 packed bytes).
  pl.tileW = (int)(W < 128 ? (W > 0 ? W : 1) : 128);
  pl.ntiles = (int)((W + pl.tileW - 1) / pl.tileW);
  if (pl.ntiles < 1) pl.ntiles = 1;
  pl.grid_x = (P4 + kThreads - 1) / kThreads;
  if (pl.grid_x < 1) pl.grid_x = 1;
  pl.smem = (size_t)pl.tileW * 16 * sizeof(double);
  return pl;
}

K2Plan k2_plan(int64_t W, int64_t P4) {
  K2Plan pl;
  pl.grid_x = (W + kThreads - 1) / kThreads;
  if (pl.grid_x < 1) pl.grid_x = 1;
  // Aim for >= ~4 CTAs per SM (148 SMs) while keeping chunks >= 64 quads.
  int64_t want_chunks = (148 * 4 + pl.grid_x - 1) / pl.grid_x;
  int64_t qc = (P4 + want_chunks - 1) / (want_chunks > 0 ? want_chunks : 1);
  if (qc < 64) qc = 64;
  if (qc > 1024) qc = 1024;
  if (qc > P4) qc = P4 > 0 ? P4 : 1;
  pl.qc = (int)qc;
  pl.nchunks = (int)((P4 + qc - 1) / qc);
  if (pl.nchunks < 1) pl.nchunks = 1;
  pl.smem = (size_t)qc * 4 * sizeof(double);
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
  k2_reduce<<<(unsigned)((g.n + 31) / 32), 256, 0, s>>>(
      zpart, kpart, pl.nchunks, g.W, g.n, g.cmiss, g.nmissing ? g.miss_col_ptr : nullptr,
      g.miss_col_idx, z);
}

}  // namespace dev
}  // namespace gkb
