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
// the full .bed information); their 3*coef contribution is removed exactly in
// the main kernels' epilogues, each CTA walking its own block's sorted
// missing list (16-bit local indices into its shared-memory coefficients).
// The reduce kernels are plain fixed-order sums of the per-CTA partials.
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

// ---------------------------------------------------------------- missing lists
// Per-CTA missing lists. The missing entries of one
// main-kernel CTA's block are stored in that block's own segment, grouped by
// the output the owning thread writes and sorted ascending, as 16-bit local
// indices:
//   K1 block (qb, tile): 128 SNP rows 4*lane+i, entries = sample offset in the tile (< 4096)
//   K2 block (wb, chunk): 512 samples 16*lane+k, entries = SNP offset in the chunk (< 2048)
// Block b's row r owns ent[base[b] + off[b*(span+1)+r] .. base[b] + off[b*(span+1)+r+1]).
// Count pass (kFill = false) writes cnt[b*span + r]; fill pass writes ent.
template <bool kFill>
__global__ void __launch_bounds__(128) k_miss_k1(const uint4* __restrict__ layA, int64_t P4,
                                                 int64_t W, int tileW, uint32_t* __restrict__ cnt,
                                                 const uint32_t* __restrict__ off,
                                                 const int64_t* __restrict__ base,
                                                 uint16_t* __restrict__ ent) {
  const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int t = threadIdx.x;  // row 4*lane + i of the K1 epilogue
  const int64_t q = (int64_t)blockIdx.x * 32 + (t >> 2);
  const int i = t & 3;
  const int64_t w0 = (int64_t)blockIdx.y * tileW, w1 = min(W, w0 + tileW);
  uint32_t c = 0;
  int64_t pos = kFill ? base[b] + off[b * 129 + t] : 0;
  if (q < P4)
    for (int64_t w = w0; w < w1; ++w) {
      const uint4 v = layA[q * W + w];
      uint32_t m = missing_mask(i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w);
      if (kFill) {
        while (m) {
          const int bit = __ffs(m) - 1;
          ent[pos++] = (uint16_t)(16 * (w - w0) + (bit >> 1));
          m &= m - 1;
        }
      } else {
        c += __popc(m);
      }
    }
  if (!kFill) cnt[b * 128 + t] = c;
}

template <bool kFill>
__global__ void __launch_bounds__(32) k_miss_k2(const uint4* __restrict__ layA, int64_t P4,
                                                int64_t W, int qc, uint32_t* __restrict__ cnt,
                                                const uint32_t* __restrict__ off,
                                                const int64_t* __restrict__ base,
                                                uint16_t* __restrict__ ent) {
  const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int lane = threadIdx.x;
  const int64_t w = (int64_t)blockIdx.x * 32 + lane;
  const int64_t q0 = (int64_t)blockIdx.y * qc, q1 = min(P4, q0 + qc);
  uint32_t c[16];
  int64_t pos[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    c[k] = 0;
    pos[k] = kFill ? base[b] + off[b * 513 + 16 * lane + k] : 0;
  }
  if (w < W)
    for (int64_t q = q0; q < q1; ++q) {
      const uint4 v = layA[q * W + w];
      const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t m = missing_mask(ws[i]);
        if (m == 0) continue;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if ((m >> (2 * k)) & 1u) {
            if (kFill)
              ent[pos[k]++] = (uint16_t)(4 * (q - q0) + i);
            else
              ++c[k];
          }
      }
    }
  if (!kFill)
#pragma unroll
    for (int k = 0; k < 16; ++k) cnt[b * 512 + 16 * lane + k] = c[k];
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
                                                    const double* __restrict__ mu,
                                                    const uint32_t* __restrict__ m_off,
                                                    const int64_t* __restrict__ m_base,
                                                    const uint16_t* __restrict__ m_ent,
                                                    double* __restrict__ ypart) {
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
  // Epilogue: thread (i, lane) owns SNP j = 4*(32*blockIdx.x + lane) + i and
  // writes this tile's exact partial
  //   sum_{observed s} r_js x_s - mu_j X_tile = sum_s r_js x_s - mu_j X_tile - (3 - mu_j) S_miss
  // with S_miss summed over the block's own missing list (scaled domain:
  // xp[s] * 2^(2(s&15)) = x_s * 2^(kS-E), exact).
  if (threadIdx.x < 128) {
    const int i = threadIdx.x >> 5;  // SNP within the quad
    const int64_t qq = (int64_t)blockIdx.x * 32 + lane;
    if (qq < P4) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += wsum[w][i][lane];
      const double m = mu[4 * qq + i];
      double v = scalbn(t, 1074 - kS + E) - m * tsum;
      if (m_off) {
        const int64_t b = (int64_t)tile * gridDim.x + blockIdx.x;
        const uint32_t* o = m_off + b * 129 + 4 * lane + i;
        const uint16_t* e = m_ent + m_base[b];
        const uint32_t e0 = o[0], e1 = o[1];
        double sm = 0.0;
        uint32_t k = e0;
        for (; k + 8 <= e1; k += 8) {  // 8 index loads in flight, summed in order
          int s[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) s[u] = e[k + u];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            sm += xp[s[u]] * __hiloint2double((1023 + 2 * (s[u] & 15)) << 20, 0);
        }
        for (; k < e1; ++k) {
          const int s1 = e[k];
          sm += xp[s1] * __hiloint2double((1023 + 2 * (s1 & 15)) << 20, 0);
        }
        if (e1 > e0) v -= (3.0 - m) * scalbn(sm, E - kS);
      }
      ypart[(int64_t)tile * 4 * P4 + 4 * qq + i] = v;
    }
  }
}

// y_j = inv_s_j * sum_t ypart[t][j]  (tiles in order -> deterministic)
__global__ void k1_reduce(const double* __restrict__ ypart, int ntiles, int64_t P4, int64_t p_loc,
                          const double* __restrict__ inv_s, double* __restrict__ y) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p_loc) return;
  double acc = 0.0;
  for (int t = 0; t < ntiles; ++t) acc += ypart[(int64_t)t * 4 * P4 + j];
  y[j] = inv_s[j] * acc;
}

// ---------------------------------------------------------------- K2 adjoint
// grid (ceil(W/32), nchunks). Lane = word position w (16 samples, 16
// accumulators); loops over the chunk's SNP quads; lanes read 32 consecutive
// 16-byte chunks of one quad row (512 B).
template <int kMinB>
__global__ void __launch_bounds__(kThreads, kMinB) k2_main(const uint4* __restrict__ layA, int64_t P4,
                                                    int64_t W, const double* __restrict__ y,
                                                    const double* __restrict__ mu,
                                                    const double* __restrict__ inv_s,
                                                    int64_t p_loc, int qc,
                                                    const uint32_t* __restrict__ m_off,
                                                    const int64_t* __restrict__ m_base,
                                                    const uint16_t* __restrict__ m_ent,
                                                    double* __restrict__ zpart) {
  // dynamic smem: cs = max(4*qc, 2048) scaled coefficients (reused for the
  // cross-warp combine), then cm = 4*qc missing-entry corrections c_j (3 - mu_j)
  extern __shared__ double2 cs2[];
  __shared__ double red[33];
  __shared__ int redi[33];
  double* cs = reinterpret_cast<double*>(cs2);
  double* cm = cs + max(4 * qc, 2048);
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
    const double m = j < p_loc ? mu[j] : 0.0;
    kp += c * m;
    if (m_off) cm[t] = c * (3.0 - m);
    cs[t] = c;
  }
  {
    const int E = block_max_int(emax, redi);
    block_sum(kp, red);  // chunk's sum_j c_j mu_j, left in red[32]
    for (int t = threadIdx.x; t < 4 * nq; t += kThreads) cs[t] = scalbn(cs[t], kS - E);
  }
  __syncthreads();

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
  // region, which is sized >= 2048 doubles). Thread (k_out, lane) owns sample
  // 16*w_out + field and writes the chunk's exact partial
  //   sum_j c_j r_js - sum_j c_j mu_j - sum_{j in miss(s)} c_j (3 - mu_j)
  // with the last sum over the block's own missing list.
  // E and ksum are re-read from shared memory (volatile: not kept live in
  // registers across the main loop, which runs at the 64-register cap)
  const int E = *reinterpret_cast<volatile int*>(&redi[32]);
  const double ksum = *reinterpret_cast<volatile double*>(&red[32]);
  double* part = cs;
  const int k_out = threadIdx.x >> 5;  // field within the half, 0..7
  const int64_t w_out = (int64_t)blockIdx.x * 32 + lane;
  double* out = zpart + (int64_t)chunk * 16 * W;
  const int64_t b = (int64_t)chunk * gridDim.x + blockIdx.x;
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
    if (w_out < W) {
      double v = scalbn(t, 1074 - kS + E - 2 * field) - ksum;
      if (m_off) {
        const uint32_t* o = m_off + b * 513 + 16 * lane + field;
        const uint16_t* e = m_ent + m_base[b];
        const uint32_t e0 = o[0], e1 = o[1];
        double corr = 0.0;
        uint32_t k = e0;
        for (; k + 8 <= e1; k += 8) {  // 8 index loads in flight, summed in order
          int jj[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) jj[u] = e[k + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) corr += cm[jj[u]];
        }
        for (; k < e1; ++k) corr += cm[e[k]];
        v -= corr;
      }
      out[16 * w_out + field] = v;
    }
  }
}

// z_s = sum_c zpart[c][s] (chunks in a fixed order -> deterministic).
// Block = 32 warps x 32 consecutive samples: warp w sums chunks c = w (mod 32)
// with lanes on consecutive samples (coalesced); partials added in warp order.
__global__ void __launch_bounds__(1024) k2_reduce(const double* __restrict__ zpart, int nchunks,
                                                  int64_t W, int64_t n, double* __restrict__ z) {
  __shared__ double part[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s = (int64_t)blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (s < n)
#pragma unroll 4
    for (int c = warp; c < nchunks; c += 32) acc += zpart[(int64_t)c * 16 * W + s];
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && s < n) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += part[w][lane];
    z[s] = t;
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

void miss_lists_k1(const uint4* layA, int64_t P4, int64_t W, const K1Plan& pl, bool fill,
                   uint32_t* cnt, const uint32_t* off, const int64_t* base, uint16_t* ent,
                   cudaStream_t s) {
  dim3 grid((unsigned)pl.grid_x, (unsigned)pl.ntiles);
  if (fill)
    k_miss_k1<true><<<grid, 128, 0, s>>>(layA, P4, W, pl.tileW, cnt, off, base, ent);
  else
    k_miss_k1<false><<<grid, 128, 0, s>>>(layA, P4, W, pl.tileW, cnt, off, base, ent);
}

void miss_lists_k2(const uint4* layA, int64_t P4, int64_t W, const K2Plan& pl, bool fill,
                   uint32_t* cnt, const uint32_t* off, const int64_t* base, uint16_t* ent,
                   cudaStream_t s) {
  dim3 grid((unsigned)pl.grid_x, (unsigned)pl.nchunks);
  if (fill)
    k_miss_k2<true><<<grid, 32, 0, s>>>(layA, P4, W, pl.qc, cnt, off, base, ent);
  else
    k_miss_k2<false><<<grid, 32, 0, s>>>(layA, P4, W, pl.qc, cnt, off, base, ent);
}

void block_scan(const uint32_t* cnt, int64_t nblk, int span, uint32_t* off, int64_t* tot,
                cudaStream_t s) {
  if (nblk == 0) return;
  k_block_scan<<<(unsigned)nblk, 512, 0, s>>>(cnt, span, off, tot);
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
  // register bound: 4 CTAs/SM (64 registers) by default; GKB_K2_MINB=3 -> 80
  const char* env = getenv("GKB_K2_MINB");
  pl.minb = (env && env[0] == '3') ? 3 : 4;
  // coefficients / combine region + missing-entry corrections
  pl.smem = (size_t)((qc * 4 > 2048 ? qc * 4 : 2048) + qc * 4) * sizeof(double);
  return pl;
}

void k1_main_only(const GenoView& g, const K1Plan& pl, const double* x, double* ypart,
                  cudaStream_t s) {
  dim3 grid((unsigned)pl.grid_x, (unsigned)pl.ntiles);
  k1_main<<<grid, kThreads, pl.smem, s>>>(g.layB, g.P4, g.W, x, g.n, pl.tileW, g.mu, g.m1_off,
                                          g.m1_base, g.m1_ent, ypart);
}

void k1_apply(const GenoView& g, const K1Plan& pl, const double* x, double* ypart, double* y,
              cudaStream_t s) {
  if (g.p_loc == 0) return;
  k1_main_only(g, pl, x, ypart, s);
  k1_reduce<<<(unsigned)((g.p_loc + 255) / 256), 256, 0, s>>>(ypart, pl.ntiles, g.P4, g.p_loc,
                                                              g.inv_s, y);
}

void k2_main_only(const GenoView& g, const K2Plan& pl, const double* y, double* zpart,
                  cudaStream_t s) {
  dim3 grid((unsigned)pl.grid_x, (unsigned)pl.nchunks);
  if (pl.minb == 3)
    k2_main<3><<<grid, kThreads, pl.smem, s>>>(g.layA, g.P4, g.W, y, g.mu, g.inv_s, g.p_loc, pl.qc,
                                               g.m2_off, g.m2_base, g.m2_ent, zpart);
  else
    k2_main<4><<<grid, kThreads, pl.smem, s>>>(g.layA, g.P4, g.W, y, g.mu, g.inv_s, g.p_loc, pl.qc,
                                               g.m2_off, g.m2_base, g.m2_ent, zpart);
}

void k2_adjoint(const GenoView& g, const K2Plan& pl, const double* y, double* zpart, double* z,
                cudaStream_t s) {
  if (g.n == 0) return;
  if (g.p_loc == 0) {
    cudaMemsetAsync(z, 0, sizeof(double) * (size_t)g.n, s);
    return;
  }
  k2_main_only(g, pl, y, zpart, s);
  k2_reduce<<<(unsigned)((g.n + 31) / 32), 1024, 0, s>>>(zpart, pl.nchunks, g.W, g.n, z);
}

}  // namespace dev
}  // namespace gkb
