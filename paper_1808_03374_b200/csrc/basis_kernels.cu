// fp64 kernels on device-resident Krylov bases (K3-K6 of SURVEY.md 2):
// tall-skinny GEMV-T/GEMV-N with fused norms (cgs2, orth.hpp:19-44), the
// structural subtraction and local second pass of partial mode
// (gkl.cpp:233-242, :277-284), thick-restart / compress recombination
// (gkl.cpp:355-359, :396-400) and the final Ritz vectors (:503-507).
//
// The products and sums that the unfused device step and the fused right tail
// (ctl_kernels.cu, compiled without contraction) must agree on are explicit
// __fma_rn / __dmul_rn (the forms the compiler contracted them to before).
//
// All of them stream a few vectors of 10^4..10^6 doubles: HBM/L2 bound and,
// at these lengths, latency bound. Each kernel therefore works on row chunks
// of kT * U rows per CTA (U rows per thread, loads of a batch issued together)
// with the CTA count near 2 per SM, and every reduction finishes inside the
// same launch: each CTA writes its partials, and the last CTA to arrive (an
// atomic ticket) sums them -- in a fixed segment order, so results are bitwise
// reproducible for a given length (the chunking is a function of the length
// only), without a second finalize launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "ctl_ops.cuh"
#include "kernels.hpp"
#include "pdl.hpp"

namespace gkb {
namespace dev {

namespace {

constexpr int kT = 256;
constexpr int kWarps = kT / 32;
constexpr int kCB = 8;      // columns per pass in gemv_t
constexpr int kBatch = 4;   // rows per thread with loads in flight together
constexpr int kSeg = 8;     // final-sum segments (one per warp)
constexpr int kTickets = 4096;  // last-CTA tickets per RedScratch

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Device-side gating (the Lanczos step control, ctl_kernels.cu): a kernel
// launched with a gate does nothing when *gate == 0 -- uniformly for all CTAs,
// so a gated-off reduction never touches its ticket.
__device__ __forceinline__ bool gated_off(const int* gate) { return gate && *gate == 0; }

// L2 load (partials written by other CTAs of this grid: skip L1)
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// After every CTA has written partial[b * K + k] (b = CTA index, k < K): the
// last CTA to arrive sums them into out[k]. Order: segment s of the nblk
// partials (fixed boundaries) summed sequentially, then the kSeg segment sums
// in order -- a function of (nblk, K) only.
// Returns true in the last CTA (all of its threads see out[]).
__device__ bool grid_finalize_cols(const double* partial, int nblk, int K, int kb, int ke,
                                   double* out, unsigned* ticket, unsigned nctas);

__device__ bool grid_finalize(const double* partial, int nblk, int K, double* out,
                              unsigned* ticket, unsigned nctas) {
  return grid_finalize_cols(partial, nblk, K, 0, K, out, ticket, nctas);
}

// Columns [kb, ke) only; `ticket` counts the nctas CTAs that write them.
__device__ bool grid_finalize_cols(const double* partial, int nblk, int K, int kb, int ke,
                                   double* out, unsigned* ticket, unsigned nctas) {
  __shared__ bool last;
  __shared__ double seg[kSeg][33];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == nctas - 1;
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = (int)((int64_t)nblk * warp / kSeg), b1 = (int)((int64_t)nblk * (warp + 1) / kSeg);
  for (int k0 = kb; k0 < ke; k0 += 32) {
    const int k = k0 + lane;
    double t = 0.0;
    if (k < ke) {
      int b = b0;
      for (; b + 4 <= b1; b += 4) {
        const double p0 = ld_cg(partial + (int64_t)b * K + k);
        const double p1 = ld_cg(partial + (int64_t)(b + 1) * K + k);
        const double p2 = ld_cg(partial + (int64_t)(b + 2) * K + k);
        const double p3 = ld_cg(partial + (int64_t)(b + 3) * K + k);
        t += p0;
        t += p1;
        t += p2;
        t += p3;
      }
      for (; b < b1; ++b) t += ld_cg(partial + (int64_t)b * K + k);
    }
    seg[warp][lane] = t;
    __syncthreads();
    if (warp == 0 && k < ke) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kSeg; ++w) s += seg[w][lane];
      out[k] = s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch on this stream
  return true;
}

// Reduces vals[0..K) across the CTA into partial[blockIdx.x * K + k] (warp
// sums, then the kWarps warp sums in order), then the grid-level finalize.
template <int K>
__device__ bool block_partial_finalize(double (&vals)[K], double* partial, double* out,
                                       unsigned* ticket) {
  __shared__ double sred[K][kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double v = warp_sum(vals[k]);
    if (lane == 0) sred[k][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) t += sred[threadIdx.x][i];
    partial[(int64_t)blockIdx.x * K + threadIdx.x] = t;
  }
  return grid_finalize(partial, gridDim.x, K, out, ticket, gridDim.x);
}

// The fused light decision (kernels.hpp ctl::Post): in the last CTA, or in
// block 0 of a gated-off launch (the decision then clears its gates).
__device__ __forceinline__ void run_post(const ctl::Post& post) {
  if (post.p.op >= 0) ctl::run_light(post.d, post.iv, post.p, threadIdx.x, blockDim.x);
}
__device__ __forceinline__ bool gated_off_post(const int* gate, const ctl::Post& post) {
  if (!gated_off(gate)) return false;
  if (blockIdx.x == 0 && blockIdx.y == 0) run_post(post);
  return true;
}

// Row chunk of CTA b: [b * rpb, min(len, (b + 1) * rpb)), rpb = kT * U.
struct Chunk {
  int64_t r0, r1;
};
__device__ __forceinline__ Chunk chunk(int64_t len, int64_t rpb) {
  Chunk c;
  c.r0 = (int64_t)blockIdx.x * rpb;
  c.r1 = min(len, c.r0 + rpb);
  return c;
}

// c[k] = Q[:, k]^T v (k < ncols), c[ncols] = ||v||^2 (with_norm). CTA (bx, by)
// covers row chunk bx and partial columns [kCB by, kCB by + kCB): kCB x kBatch
// independent loads per thread in flight, warp sums per column, then the
// kWarps warp sums in order into partial[bx * K + k].
// kBatchT rows per thread per batch (x kCB columns of loads in flight): a
// thread visits the same rows in the same order for any batch size, so the
// sums do not depend on it -- 4 for one-group calls (few columns), else 2
// (registers: 76 instead of 116).
template <int kBatchT>
__global__ void __launch_bounds__(kT) k_gemv_t(const double* __restrict__ Q, int64_t ld,
                                               int64_t len, int64_t ncols,
                                               const double* __restrict__ v, int with_norm,
                                               int64_t rpb, int K, double* __restrict__ partial,
                                               double* __restrict__ out,
                                               unsigned* __restrict__ ticket, const int* gate) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  __shared__ double ws[kCB][kWarps];
  if (gated_off(gate)) return;
  const Chunk ch = chunk(len, rpb);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.y * kCB;
  double acc[kCB];
#pragma unroll
  for (int k = 0; k < kCB; ++k) acc[k] = 0.0;
  for (int64_t rb = ch.r0 + threadIdx.x; rb < ch.r1; rb += (int64_t)kT * kBatchT) {
    double vr[kBatchT];
#pragma unroll
    for (int i = 0; i < kBatchT; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      vr[i] = r < ch.r1 ? v[r] : 0.0;
    }
    // all kCB x kBatchT loads issued before the FMAs (as in k_gemv_n): the
    // FMA order per column is unchanged, so are the bits
    double q[kCB][kBatchT];
#pragma unroll
    for (int k = 0; k < kCB; ++k) {
      const int64_t c = c0 + k;
#pragma unroll
      for (int i = 0; i < kBatchT; ++i) {
        const int64_t r = rb + (int64_t)i * kT;
        q[k][i] = (c < ncols && r < ch.r1) ? Q[c * ld + r] : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kCB; ++k) {
      const int64_t c = c0 + k;
      if (c < ncols) {
#pragma unroll
        for (int i = 0; i < kBatchT; ++i) {
          const int64_t r = rb + (int64_t)i * kT;
          if (r < ch.r1) acc[k] = __fma_rn(q[k][i], vr[i], acc[k]);
        }
      } else if (c == ncols && with_norm) {
#pragma unroll
        for (int i = 0; i < kBatchT; ++i) acc[k] = __fma_rn(vr[i], vr[i], acc[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kCB; ++k) {
    const double t = warp_sum(acc[k]);
    if (lane == 0) ws[k][warp] = t;
  }
  __syncthreads();
  if (threadIdx.x < kCB && c0 + threadIdx.x < K) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += ws[threadIdx.x][w];
    partial[(int64_t)blockIdx.x * K + c0 + threadIdx.x] = t;
  }
  // the last row chunk of this column group sums its kCB columns (one ticket
  // per group: the groups finish in parallel, same per-column order)
  grid_finalize_cols(partial, gridDim.x, K, (int)c0, (int)min((int64_t)K, c0 + kCB), out,
                     ticket + blockIdx.y, gridDim.x);
}

// v = beta*v + sign*(Q c); optional norms before/after (out[0], out[1]).
__global__ void __launch_bounds__(kT) k_gemv_n(const double* __restrict__ Q, int64_t ld,
                                               int64_t len, int64_t ncols,
                                               const double* __restrict__ c,
                                               double* __restrict__ v, double beta, double sign,
                                               int norms, int64_t rpb,
                                               double* __restrict__ partial,
                                               double* __restrict__ out,
                                               unsigned* __restrict__ ticket, const int* gate,
                                               const ctl::Post post) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  __shared__ double cs[1024];
  if (gated_off_post(gate, post)) return;
  const Chunk ch = chunk(len, rpb);
  double nrm[2] = {0.0, 0.0};
  for (int64_t rb = ch.r0 + threadIdx.x; rb - threadIdx.x < ch.r1; rb += (int64_t)kT * kBatch) {
    double s[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) s[i] = 0.0;
    for (int64_t cb = 0; cb < ncols; cb += 1024) {
      const int64_t cn = min((int64_t)1024, ncols - cb);
      __syncthreads();
      for (int t = threadIdx.x; t < cn; t += kT) cs[t] = c[cb + t];
      __syncthreads();
      int64_t l = 0;
      for (; l + kCB <= cn; l += kCB) {  // kCB columns x kBatch rows of loads in flight
        double q[kCB][kBatch];
#pragma unroll
        for (int k = 0; k < kCB; ++k)
#pragma unroll
          for (int i = 0; i < kBatch; ++i) {
            const int64_t r = rb + (int64_t)i * kT;
            q[k][i] = r < ch.r1 ? Q[(cb + l + k) * ld + r] : 0.0;
          }
#pragma unroll
        for (int k = 0; k < kCB; ++k)
#pragma unroll
          for (int i = 0; i < kBatch; ++i) s[i] = __fma_rn(q[k][i], cs[l + k], s[i]);
      }
      for (; l < cn; ++l) {
        const double* q0 = Q + (cb + l) * ld;
        const double w0 = cs[l];
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
          const int64_t r = rb + (int64_t)i * kT;
          if (r < ch.r1) s[i] = __fma_rn(q0[r], w0, s[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      if (r < ch.r1) {
        const double old = v[r];
        const double nv = beta == 0.0 ? __dmul_rn(sign, s[i])
                                      : __fma_rn(beta, old, __dmul_rn(sign, s[i]));
        v[r] = nv;
        nrm[0] = __fma_rn(old, old, nrm[0]);
        nrm[1] = __fma_rn(nv, nv, nrm[1]);
      }
    }
  }
  if (norms && block_partial_finalize<2>(nrm, partial, out, ticket)) run_post(post);
}

__global__ void __launch_bounds__(kT) k_dot(const double* __restrict__ a,
                                            const double* __restrict__ b, int64_t len,
                                            int64_t rpb, double* __restrict__ partial,
                                            double* __restrict__ out,
                                            unsigned* __restrict__ ticket, const int* gate,
                                            const ctl::Post post) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  if (gated_off_post(gate, post)) return;
  const Chunk ch = chunk(len, rpb);
  double acc[1] = {0.0};
  for (int64_t rb = ch.r0 + threadIdx.x; rb < ch.r1; rb += (int64_t)kT * kBatch) {
    double x[kBatch], y[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      x[i] = r < ch.r1 ? a[r] : 0.0;
      y[i] = r < ch.r1 ? b[r] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) acc[0] = __fma_rn(x[i], y[i], acc[0]);
  }
  if (block_partial_finalize<1>(acc, partial, out, ticket)) run_post(post);
}

// v -= (*dprev) * uprev (when `uprev` is set and agate is on), then
// out[0] = sum unext * v (v itself when unext is null) when dgate is on: one
// step of the sequential local second pass (gkl.cpp:233-242, :277-284) with
// the next column's dot, or the final norm, in the same pass. Same chunking,
// products and sum order as k_axpy_dev followed by k_dot, so the same bits.
__global__ void __launch_bounds__(kT) k_axpy_dot(const double* __restrict__ dprev,
                                                 const double* __restrict__ uprev,
                                                 const int* agate,
                                                 const double* __restrict__ unext,
                                                 const int* dgate, double* __restrict__ v,
                                                 int64_t len, int64_t rpb,
                                                 double* __restrict__ partial,
                                                 double* __restrict__ out,
                                                 unsigned* __restrict__ ticket) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  const bool aon = uprev != nullptr && !gated_off(agate);
  const bool don = !gated_off(dgate);
  if (!aon && !don) return;
  const double a = aon ? *dprev : 0.0;
  const Chunk ch = chunk(len, rpb);
  double acc[1] = {0.0};
  for (int64_t rb = ch.r0 + threadIdx.x; rb < ch.r1; rb += (int64_t)kT * kBatch) {
    double x[kBatch], y[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      x[i] = r < ch.r1 ? v[r] : 0.0;
      y[i] = (aon && r < ch.r1) ? uprev[r] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      if (aon && r < ch.r1) {
        x[i] = __fma_rn(-a, y[i], x[i]);
        v[r] = x[i];
      }
    }
    if (don) {
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int64_t r = rb + (int64_t)i * kT;
        y[i] = unext ? (r < ch.r1 ? unext[r] : 0.0) : x[i];
      }
#pragma unroll
      for (int i = 0; i < kBatch; ++i) acc[0] = __fma_rn(y[i], x[i], acc[0]);
    }
  }
  if (don) block_partial_finalize<1>(acc, partial, out, ticket);
}

// sum (a - b)^2 (subspace delta criterion)
__global__ void __launch_bounds__(kT) k_diff_nrm2(const double* __restrict__ a,
                                                  const double* __restrict__ b, int64_t len,
                                                  int64_t rpb, double* __restrict__ partial,
                                                  double* __restrict__ out,
                                                  unsigned* __restrict__ ticket) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  const Chunk ch = chunk(len, rpb);
  double acc[1] = {0.0};
  for (int64_t rb = ch.r0 + threadIdx.x; rb < ch.r1; rb += (int64_t)kT * kBatch) {
    double d[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      d[i] = r < ch.r1 ? a[r] - b[r] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) acc[0] += d[i] * d[i];
  }
  block_partial_finalize<1>(acc, partial, out, ticket);
}

__global__ void k_axpy_dev(const double* __restrict__ d, const double* __restrict__ u,
                           double* __restrict__ v, int64_t len, const int* gate) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  if (gated_off(gate)) return;
  const double a = *d;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < len;
       r += (int64_t)gridDim.x * blockDim.x)
    v[r] -= a * u[r];
}

// v = v - alpha*u with ||v_before||^2, ||v_after||^2. alpha is the host value,
// or read on the device from `dval`: sqrt(*dval) (take_sqrt; IEEE sqrt, bitwise
// equal to the host's std::sqrt of the same value) or *dval itself.
__global__ void __launch_bounds__(kT) k_axpy_norms(double alpha, const double* __restrict__ dval,
                                                   int take_sqrt, const double* __restrict__ u,
                                                   double* __restrict__ v, int64_t len,
                                                   int64_t rpb, double* __restrict__ partial,
                                                   double* __restrict__ out,
                                                   unsigned* __restrict__ ticket, const int* gate,
                                                   const ctl::Post post) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  if (gated_off_post(gate, post)) return;
  if (dval) alpha = take_sqrt ? sqrt(*dval) : *dval;
  const Chunk ch = chunk(len, rpb);
  double acc[2] = {0.0, 0.0};
  for (int64_t rb = ch.r0 + threadIdx.x; rb < ch.r1; rb += (int64_t)kT * kBatch) {
    double x[kBatch], y[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      x[i] = r < ch.r1 ? v[r] : 0.0;
      y[i] = r < ch.r1 ? u[r] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int64_t r = rb + (int64_t)i * kT;
      const double nv = __fma_rn(-alpha, y[i], x[i]);
      if (r < ch.r1) v[r] = nv;
      acc[0] = __fma_rn(x[i], x[i], acc[0]);
      acc[1] = __fma_rn(nv, nv, acc[1]);
    }
  }
  if (block_partial_finalize<2>(acc, partial, out, ticket)) run_post(post);
}

__global__ void k_div_copy_dev(const double* __restrict__ src, const double* __restrict__ dval,
                               int take_sqrt, double* __restrict__ dst, int64_t len,
                               const int* gate) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  if (gated_off(gate)) return;
  const double divisor = take_sqrt ? sqrt(*dval) : *dval;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < len;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[r] / divisor;
}

__global__ void k_div_copy(const double* __restrict__ src, double divisor, double* __restrict__ dst,
                           int64_t len) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < len;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[r] / divisor;
}

// dst[:, c] = sum_l Q[:, l] * W[l, c] for c in [c0, c0 + NC): one row per
// thread, Q read once per pass of NC output columns, W staged in smem.
template <int NC>
__global__ void __launch_bounds__(128) k_gemm_small(const double* __restrict__ Q, int64_t ld,
                                                    int64_t len, int64_t j,
                                                    const double* __restrict__ W, int64_t ldw,
                                                    int64_t kc, int64_t c0,
                                                    double* __restrict__ dst, int64_t ldd) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  extern __shared__ double wsm[];  // j x NC
  for (int64_t t = threadIdx.x; t < j * NC; t += blockDim.x) {
    const int64_t l = t / NC, c = c0 + t % NC;
    wsm[t] = c < kc ? W[c * ldw + l] : 0.0;
  }
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= len) return;
  double acc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) acc[k] = 0.0;
  int64_t l = 0;
  for (; l + 4 <= j; l += 4) {
    double q[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = Q[(l + i) * ld + r];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < NC; ++k) acc[k] += q[i] * wsm[(l + i) * NC + k];
  }
  for (; l < j; ++l) {
    const double q = Q[l * ld + r];
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] += q * wsm[l * NC + k];
  }
#pragma unroll
  for (int k = 0; k < NC; ++k)
    if (c0 + k < kc) dst[(c0 + k) * ldd + r] = acc[k];
}

struct SrcList {
  const double* p[16];
};

__global__ void k_sum_buffers(SrcList l, int nsrc, double* __restrict__ dst, int64_t len) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
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

// rows per thread: enough CTAs for ~2 per SM, at most 64 rows per thread
int64_t rows_per_thread(int64_t len) {
  int64_t u = (len + (int64_t)kT * 296 - 1) / ((int64_t)kT * 296);
  if (u < 1) u = 1;
  if (u > 64) u = 64;
  return u;
}

int64_t rpb_of(int64_t len) { return (int64_t)kT * rows_per_thread(len); }

// gemv_t / gemv_n row chunking (their partials are their own, so it may differ
// from the other reductions'): about `blocks` row chunks (GKB_GT_BLOCKS,
// GKB_GN_BLOCKS for sweeps)
int64_t rpb_target(int64_t len, const char* env, int64_t dflt) {
  int64_t blocks = dflt;
  if (const char* e = getenv(env)) blocks = std::max<int64_t>(1, atoll(e));
  int64_t u = (len + (int64_t)kT * blocks - 1) / ((int64_t)kT * blocks);
  if (u < 1) u = 1;
  if (u > 256) u = 256;
  return (int64_t)kT * u;
}

}  // namespace

int64_t red_blocks(int64_t len) {
  // a function of len only (determinism)
  const int64_t rpb = rpb_of(len);
  const int64_t b = (len + rpb - 1) / rpb;
  return b > 0 ? b : 1;
}

namespace {
ctl::Post post_of(const ctl::Post* p) {
  if (p) return *p;
  ctl::Post none;
  none.p.op = -1;
  return none;
}

}  // namespace

void init_red_scratch(RedScratch& rs) {
  if (!rs.ticket) {  // one per gemv_t column group (K <= 8 * kTickets), [0] for the rest
    cudaMalloc(&rs.ticket, sizeof(unsigned) * kTickets);
    cudaMemset(rs.ticket, 0, sizeof(unsigned) * kTickets);
  }
}

void gemv_t(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* v, bool with_norm,
            RedScratch& rs, double* out, cudaStream_t s, const int* gate) {
  const int K = (int)(ncols + (with_norm ? 1 : 0));
  if (K == 0) return;
  if ((K + kCB - 1) / kCB > kTickets) {  // (beyond 32K columns: column blocks of 32K)
    for (int64_t c0 = 0; c0 < ncols; c0 += 8 * (int64_t)kTickets) {
      const int64_t cn = std::min<int64_t>(8 * (int64_t)kTickets, ncols - c0);
      const bool nrm = with_norm && c0 + cn == ncols;
      gemv_t(Q + c0 * ld, ld, len, cn, v, nrm, rs, out + c0, s, gate);
    }
    return;
  }
  // row chunks: ~74 (below 300k rows) / 148 (basis_bench sweep: 100k x 50
  // 14.4 -> 10.6 us, 500k x 50 46.7 -> 43.3 us against 296); at most 18,944
  // rows stay 256-row chunks (the fused right tail reduces like these CTAs)
  const int64_t rpb = rpb_target(len, "GKB_GT_BLOCKS", len < 300000 ? 74 : 148);
  const int64_t nb = std::max<int64_t>(1, (len + rpb - 1) / rpb);
  const dim3 grid((unsigned)nb, (unsigned)((K + kCB - 1) / kCB));
  launch_pdl(K <= 4 ? k_gemv_t<4> : k_gemv_t<2>, grid, dim3(kT), 0, s, true, Q, ld, len, ncols, v,
             with_norm ? 1 : 0, rpb, K, rs.partial, out, rs.ticket, gate);
}

void gemv_n(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* c, double* v,
            double beta, double sign, bool norms, RedScratch& rs, double* out, cudaStream_t s,
            const int* gate, const ctl::Post* post) {
  if (len == 0 && !norms) return;
  // ~148 row chunks below 300k rows (100k x 50: 9.9 -> 8.5 us), 296 above
  const int64_t rpb = rpb_target(len, "GKB_GN_BLOCKS", len < 300000 ? 148 : 296);
  const int64_t nb = std::max<int64_t>(1, (len + rpb - 1) / rpb);
  launch_pdl(k_gemv_n, dim3((unsigned)nb), dim3(kT), 0, s, true, Q, ld, len, ncols, c, v, beta,
             sign, norms ? 1 : 0, rpb, rs.partial, out, rs.ticket, gate, post_of(post));
}

void dot(const double* a, const double* b, int64_t len, RedScratch& rs, double* out, cudaStream_t s,
         const int* gate, const ctl::Post* post) {
  launch_pdl(k_dot, dim3((unsigned)red_blocks(len)), dim3(kT), 0, s, true, a, b, len, rpb_of(len),
             rs.partial, out, rs.ticket, gate, post_of(post));
}

void nrm2sq(const double* a, int64_t len, RedScratch& rs, double* out, cudaStream_t s,
            const int* gate, const ctl::Post* post) {
  dot(a, a, len, rs, out, s, gate, post);
}

void axpy_dot(const double* dprev, const double* uprev, const int* agate, const double* unext,
              const int* dgate, double* v, int64_t len, RedScratch& rs, double* out,
              cudaStream_t s) {
  launch_pdl(k_axpy_dot, dim3((unsigned)red_blocks(len)), dim3(kT), 0, s, true, dprev, uprev, agate,
             unext, dgate, v, len, rpb_of(len), rs.partial, out, rs.ticket);
}

void diff_nrm2sq(const double* a, const double* b, int64_t len, RedScratch& rs, double* out,
                 cudaStream_t s) {
  launch_pdl(k_diff_nrm2, dim3((unsigned)red_blocks(len)), dim3(kT), 0, s, true, a, b, len,
             rpb_of(len), rs.partial, out, rs.ticket);
}

void axpy_dev(const double* dptr, const double* u, double* v, int64_t len, cudaStream_t s,
              const int* gate) {
  if (len == 0) return;
  launch_pdl(k_axpy_dev, dim3(elem_grid(len)), dim3(kT), 0, s, true, dptr, u, v, len, gate);
}

void axpy_norms(double alpha, const double* u, double* v, int64_t len, RedScratch& rs, double* out,
                cudaStream_t s) {
  launch_pdl(k_axpy_norms, dim3((unsigned)red_blocks(len)), dim3(kT), 0, s, true, alpha, nullptr, 0, u, v, len,
             rpb_of(len), rs.partial, out, rs.ticket, nullptr, post_of(nullptr));
}

void axpy_norms_dsq(const double* nrm2, const double* u, double* v, int64_t len, RedScratch& rs,
                    double* out, cudaStream_t s) {
  launch_pdl(k_axpy_norms, dim3((unsigned)red_blocks(len)), dim3(kT), 0, s, true, 0.0, nrm2, 1, u, v, len, rpb_of(len),
             rs.partial, out, rs.ticket, nullptr, post_of(nullptr));
}

void axpy_norms_dv(const double* alpha, const double* u, double* v, int64_t len, RedScratch& rs,
                   double* out, cudaStream_t s, const int* gate, const ctl::Post* post) {
  launch_pdl(k_axpy_norms, dim3((unsigned)red_blocks(len)), dim3(kT), 0, s, true, 0.0, alpha, 0, u, v, len, rpb_of(len),
             rs.partial, out, rs.ticket, gate, post_of(post));
}

void div_copy_dsq(const double* src, const double* nrm2, double* dst, int64_t len,
                  cudaStream_t s) {
  if (len == 0) return;
  launch_pdl(k_div_copy_dev, dim3(elem_grid(len)), dim3(kT), 0, s, true, src, nrm2, 1, dst, len, nullptr);
}

void div_copy_dv(const double* src, const double* divisor, double* dst, int64_t len,
                 cudaStream_t s, const int* gate) {
  if (len == 0) return;
  launch_pdl(k_div_copy_dev, dim3(elem_grid(len)), dim3(kT), 0, s, true, src, divisor, 0, dst, len, gate);
}

void div_copy(const double* src, double divisor, double* dst, int64_t len, cudaStream_t s) {
  if (len == 0) return;
  launch_pdl(k_div_copy, dim3(elem_grid(len)), dim3(kT), 0, s, true, src, divisor, dst, len);
}

void gemm_small(const double* Q, int64_t ld, int64_t len, int64_t j, const double* W, int64_t ldw,
                int64_t kc, double* dst, int64_t ldd, cudaStream_t s) {
  if (len == 0 || kc == 0) return;
  const unsigned grid = (unsigned)((len + 127) / 128);
  for (int64_t c0 = 0; c0 < kc; c0 += 32) {
    const int64_t rem = kc - c0;
    if (rem > 16) {
      const size_t sm = sizeof(double) * (size_t)(j * 32);
      if (sm > 48 * 1024)
        cudaFuncSetAttribute(k_gemm_small<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
      launch_pdl(k_gemm_small<32>, grid, dim3(128), sm, s, true, Q, ld, len, j, W, ldw, kc, c0, dst, ldd);
    } else if (rem > 8) {
      launch_pdl(k_gemm_small<16>, grid, dim3(128), sizeof(double) * (size_t)(j * 16), s, true, Q, ld, len, j, W, ldw,
                                                                            kc, c0, dst, ldd);
    } else {
      launch_pdl(k_gemm_small<8>, grid, dim3(128), sizeof(double) * (size_t)(j * 8), s, true, Q, ld, len, j, W, ldw,
                                                                          kc, c0, dst, ldd);
    }
  }
}

void sum_buffers(const double* const* srcs, int nsrc, double* dst, int64_t len, cudaStream_t s) {
  SrcList l;
  for (int k = 0; k < 16; ++k) l.p[k] = k < nsrc ? srcs[k] : nullptr;
  if (len == 0) return;
  launch_pdl(k_sum_buffers, dim3(elem_grid(len)), dim3(kT), 0, s, true, l, nsrc, dst, len);
}

void flush_l2(void* buf, size_t bytes, cudaStream_t s) { cudaMemsetAsync(buf, 0, bytes, s); }

}  // namespace dev
}  // namespace gkb
