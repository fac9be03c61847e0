// fp64 kernels on device-resident Krylov bases (K3-K6 of SURVEY.md 2):
// tall-skinny GEMV-T/GEMV-N with fused norms (cgs2, orth.hpp:19-44), the
// structural subtraction and local second pass of partial mode
// (gkl.cpp:233-242, :277-284), thick-restart / compress recombination
// (gkl.cpp:355-359, :396-400) and the final Ritz vectors (:503-507).
//
// Every reduction writes per-block partials and a one-block finalize sums
// them in block order, so results are bitwise reproducible for a given
// length (the block count is a function of the length only).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace gkb {
namespace dev {

namespace {

constexpr int kT = 256;
constexpr int kCB = 8;  // columns per CTA in gemv_t

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Reduces vals[0..K) across the block; thread 0 writes out[k].
template <int K>
__device__ void block_reduce_write(double (&vals)[K], double* out) {
  __shared__ double sred[K][kT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double v = warp_sum(vals[k]);
    if (lane == 0) sred[k][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double t = 0.0;
    for (int i = 0; i < kT / 32; ++i) t += sred[threadIdx.x][i];
    out[threadIdx.x] = t;
  }
}

__global__ void k_gemv_t(const double* __restrict__ Q, int64_t ld, int64_t len, int64_t ncols,
                         const double* __restrict__ v, int with_norm, int64_t rows_per_block,
                         int K, double* __restrict__ partial) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(len, r0 + rows_per_block);
  const int64_t c0 = (int64_t)blockIdx.y * kCB;
  double acc[kCB + 1];
#pragma unroll
  for (int k = 0; k <= kCB; ++k) acc[k] = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kT) {
    const double vr = v[r];
#pragma unroll
    for (int k = 0; k < kCB; ++k)
      if (c0 + k < ncols) acc[k] += Q[(c0 + k) * ld + r] * vr;
    acc[kCB] += vr * vr;
  }
  __shared__ double outv[kCB + 1];
  block_reduce_write<kCB + 1>(acc, outv);
  __syncthreads();
  if (threadIdx.x < kCB + 1) {
    const int k = threadIdx.x;
    if (k < kCB && c0 + k < ncols) partial[(int64_t)blockIdx.x * K + c0 + k] = outv[k];
    if (k == kCB && with_norm && blockIdx.y == 0) partial[(int64_t)blockIdx.x * K + ncols] = outv[k];
  }
}

// out[k] = sum_b partial[b*K + k]
__global__ void k_finalize(const double* __restrict__ partial, int nblk, int K,
                           double* __restrict__ out) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double t = 0.0;
    for (int b = 0; b < nblk; ++b) t += partial[(int64_t)b * K + k];
    out[k] = t;
  }
}

// v = beta*v + sign*(Q c); optional norms before/after into block partials
__global__ void k_gemv_n(const double* __restrict__ Q, int64_t ld, int64_t len, int64_t ncols,
                         const double* __restrict__ c, double* __restrict__ v, double beta,
                         double sign, int norms, int64_t rows_per_block,
                         double* __restrict__ partial) {
  __shared__ double cs[1024];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(len, r0 + rows_per_block);
  double acc2[2] = {0.0, 0.0};
  // rows handled by this thread: r0 + threadIdx.x + i*kT
  for (int64_t rb = r0; rb < r1; rb += kT) {
    const int64_t r = rb + threadIdx.x;
    double s = 0.0;
    for (int64_t cb = 0; cb < ncols; cb += 1024) {
      const int64_t cn = min((int64_t)1024, ncols - cb);
      __syncthreads();
      for (int t = threadIdx.x; t < cn; t += kT) cs[t] = c[cb + t];
      __syncthreads();
      if (r < r1)
        for (int64_t l = 0; l < cn; ++l) s += Q[(cb + l) * ld + r] * cs[l];
    }
    if (r < r1) {
      const double old = v[r];
      const double nv = beta == 0.0 ? sign * s : beta * old + sign * s;
      v[r] = nv;
      acc2[0] += old * old;
      acc2[1] += nv * nv;
    }
  }
  if (norms) block_reduce_write<2>(acc2, partial + (int64_t)blockIdx.x * 2);
}

__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t len,
                      int64_t rows_per_block, double* __restrict__ partial) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(len, r0 + rows_per_block);
  double acc[1] = {0.0};
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kT) acc[0] += a[r] * b[r];
  block_reduce_write<1>(acc, partial + blockIdx.x);
}

__global__ void k_axpy_dev(const double* __restrict__ d, const double* __restrict__ u,
                           double* __restrict__ v, int64_t len) {
  const double a = *d;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < len;
       r += (int64_t)gridDim.x * blockDim.x)
    v[r] -= a * u[r];
}

__global__ void k_axpy_norms(double alpha, const double* __restrict__ u, double* __restrict__ v,
                             int64_t len, int64_t rows_per_block, double* __restrict__ partial) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(len, r0 + rows_per_block);
  double acc[2] = {0.0, 0.0};
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kT) {
    const double old = v[r];
    const double nv = old - alpha * u[r];
    v[r] = nv;
    acc[0] += old * old;
    acc[1] += nv * nv;
  }
  block_reduce_write<2>(acc, partial + (int64_t)blockIdx.x * 2);
}

// alpha = sqrt(*nrm2) read on the device (IEEE sqrt: bitwise equal to the
// host's std::sqrt of the same value) -- used to launch the next half-step
// before the host has read the norm.
__global__ void k_axpy_norms_dsq(const double* __restrict__ nrm2, const double* __restrict__ u,
                                 double* __restrict__ v, int64_t len, int64_t rows_per_block,
                                 double* __restrict__ partial) {
  const double alpha = sqrt(*nrm2);
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(len, r0 + rows_per_block);
  double acc[2] = {0.0, 0.0};
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kT) {
    const double old = v[r];
    const double nv = old - alpha * u[r];
    v[r] = nv;
    acc[0] += old * old;
    acc[1] += nv * nv;
  }
  block_reduce_write<2>(acc, partial + (int64_t)blockIdx.x * 2);
}

__global__ void k_div_copy_dsq(const double* __restrict__ src, const double* __restrict__ nrm2,
                               double* __restrict__ dst, int64_t len) {
  const double divisor = sqrt(*nrm2);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < len;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[r] / divisor;
}

__global__ void k_div_copy(const double* __restrict__ src, double divisor, double* __restrict__ dst,
                           int64_t len) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < len;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[r] / divisor;
}

// dst[:, c] = sum_l Q[:, l] * W[l, c], 8 output columns per pass
__global__ void k_gemm_small(const double* __restrict__ Q, int64_t ld, int64_t len, int64_t j,
                             const double* __restrict__ W, int64_t ldw, int64_t kc,
                             double* __restrict__ dst, int64_t ldd) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= len) return;
  for (int64_t c0 = 0; c0 < kc; c0 += 8) {
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
    for (int64_t l = 0; l < j; ++l) {
      const double q = Q[l * ld + r];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + k < kc) acc[k] += q * __ldg(W + (c0 + k) * ldw + l);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c0 + k < kc) dst[(c0 + k) * ldd + r] = acc[k];
  }
}

struct SrcList {
  const double* p[16];
};

__global__ void k_sum_buffers(SrcList l, int nsrc, double* __restrict__ dst, int64_t len) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < len;
       r += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int k = 0; k < nsrc; ++k) t += l.p[k][r];
    dst[r] = t;
  }
}

int elem_grid(int64_t len) {
  int64_t g = (len + kT - 1) / kT;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  return (int)g;
}

int64_t rows_per_block(int64_t len, int64_t nblk) {
  int64_t rpb = (len + nblk - 1) / nblk;
  rpb = ((rpb + kT - 1) / kT) * kT;
  return rpb > 0 ? rpb : kT;
}

}  // namespace

int64_t red_blocks(int64_t len) {
  // function of len only (determinism); ~4 rows per thread, at most 296 blocks
  int64_t b = (len + kT * 4 - 1) / (kT * 4);
  if (b > 296) b = 296;
  if (b < 1) b = 1;
  return b;
}

void gemv_t(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* v, bool with_norm,
            RedScratch& rs, double* out, cudaStream_t s) {
  const int K = (int)(ncols + (with_norm ? 1 : 0));
  if (K == 0) return;
  const int64_t nb = red_blocks(len);
  const int64_t rpb = rows_per_block(len, nb);
  const int64_t nblk = (len + rpb - 1) / rpb > 0 ? (len + rpb - 1) / rpb : 1;
  const int64_t cb = ncols > 0 ? (ncols + kCB - 1) / kCB : 1;
  k_gemv_t<<<dim3((unsigned)nblk, (unsigned)cb), kT, 0, s>>>(Q, ld, len, ncols, v, with_norm ? 1 : 0,
                                                            rpb, K, rs.partial);
  k_finalize<<<1, 256, 0, s>>>(rs.partial, (int)nblk, K, out);
}

void gemv_n(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* c, double* v,
            double beta, double sign, bool norms, RedScratch& rs, double* out, cudaStream_t s) {
  const int64_t nb = red_blocks(len);
  const int64_t rpb = rows_per_block(len, nb);
  const int64_t nblk = (len + rpb - 1) / rpb > 0 ? (len + rpb - 1) / rpb : 1;
  k_gemv_n<<<(unsigned)nblk, kT, 0, s>>>(Q, ld, len, ncols, c, v, beta, sign, norms ? 1 : 0, rpb,
                                         rs.partial);
  if (norms) k_finalize<<<1, 32, 0, s>>>(rs.partial, (int)nblk, 2, out);
}

void dot(const double* a, const double* b, int64_t len, RedScratch& rs, double* out, cudaStream_t s) {
  const int64_t nb = red_blocks(len);
  const int64_t rpb = rows_per_block(len, nb);
  const int64_t nblk = (len + rpb - 1) / rpb > 0 ? (len + rpb - 1) / rpb : 1;
  k_dot<<<(unsigned)nblk, kT, 0, s>>>(a, b, len, rpb, rs.partial);
  k_finalize<<<1, 32, 0, s>>>(rs.partial, (int)nblk, 1, out);
}

void nrm2sq(const double* a, int64_t len, RedScratch& rs, double* out, cudaStream_t s) {
  dot(a, a, len, rs, out, s);
}

void axpy_dev(const double* dptr, const double* u, double* v, int64_t len, cudaStream_t s) {
  if (len == 0) return;
  k_axpy_dev<<<elem_grid(len), kT, 0, s>>>(dptr, u, v, len);
}

void axpy_norms(double alpha, const double* u, double* v, int64_t len, RedScratch& rs, double* out,
                cudaStream_t s) {
  const int64_t nb = red_blocks(len);
  const int64_t rpb = rows_per_block(len, nb);
  const int64_t nblk = (len + rpb - 1) / rpb > 0 ? (len + rpb - 1) / rpb : 1;
  k_axpy_norms<<<(unsigned)nblk, kT, 0, s>>>(alpha, u, v, len, rpb, rs.partial);
  k_finalize<<<1, 32, 0, s>>>(rs.partial, (int)nblk, 2, out);
}

void axpy_norms_dsq(const double* nrm2, const double* u, double* v, int64_t len, RedScratch& rs,
                    double* out, cudaStream_t s) {
  const int64_t nb = red_blocks(len);
  const int64_t rpb = rows_per_block(len, nb);
  const int64_t nblk = (len + rpb - 1) / rpb > 0 ? (len + rpb - 1) / rpb : 1;
  k_axpy_norms_dsq<<<(unsigned)nblk, kT, 0, s>>>(nrm2, u, v, len, rpb, rs.partial);
  k_finalize<<<1, 32, 0, s>>>(rs.partial, (int)nblk, 2, out);
}

void div_copy_dsq(const double* src, const double* nrm2, double* dst, int64_t len,
                  cudaStream_t s) {
  if (len == 0) return;
  k_div_copy_dsq<<<elem_grid(len), kT, 0, s>>>(src, nrm2, dst, len);
}

void div_copy(const double* src, double divisor, double* dst, int64_t len, cudaStream_t s) {
  if (len == 0) return;
  k_div_copy<<<elem_grid(len), kT, 0, s>>>(src, divisor, dst, len);
}

void gemm_small(const double* Q, int64_t ld, int64_t len, int64_t j, const double* W, int64_t ldw,
                int64_t kc, double* dst, int64_t ldd, cudaStream_t s) {
  if (len == 0 || kc == 0) return;
  k_gemm_small<<<(unsigned)((len + 127) / 128), 128, 0, s>>>(Q, ld, len, j, W, ldw, kc, dst, ldd);
}

void sum_buffers(const double* const* srcs, int nsrc, double* dst, int64_t len, cudaStream_t s) {
  SrcList l;
  for (int k = 0; k < 16; ++k) l.p[k] = k < nsrc ? srcs[k] : nullptr;
  if (len == 0) return;
  k_sum_buffers<<<elem_grid(len), kT, 0, s>>>(l, nsrc, dst, len);
}

void flush_l2(void* buf, size_t bytes, cudaStream_t s) { cudaMemsetAsync(buf, 0, bytes, s); }

}  // namespace dev
}  // namespace gkb
