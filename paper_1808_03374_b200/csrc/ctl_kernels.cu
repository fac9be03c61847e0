// Device-side step control of the GKL bidiagonalization.
//
// The host-driven step (gkl_driver.cpp, Lanczos::step) reads norms back after
// every reduction to take the reference's decisions: the local second pass
// (gkl.cpp:233-242, :277-284), the omega recurrences and the reorthogonalize
// test (partial_reorth_update, gkl.cpp:112-176), the cgs2 second pass
// (orth.hpp:30-41) and the breakdown tests (gkl.cpp:246, :292). Here the same
// decisions are taken by one small CTA on the device, from the same device
// scalars, and written to int gates that the following kernels test before
// doing anything (kernels.hpp: `gate`). The host can then enqueue a whole
// restart cycle of steps without reading anything back.
//
// Every expression follows the host code's operation order, and this file is
// compiled with -fmad=false (no FMA contraction, like the host's
// -ffp-contract=off), so the recurrences produce the host path's bits. The
// one exception is hypot in the norm-scale update (CUDA's hypot may differ
// from the C library's in the last place); norm_scale only enters tau and
// the breakdown threshold.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.hpp"
#include "pdl.hpp"
#include "ctl_ops.cuh"

namespace gkb {
namespace dev {
namespace ctl {

namespace {

constexpr int kCtlThreads = 128;

__device__ void run_op(double* __restrict__ d, int* __restrict__ iv, const Params& p) {
  const Layout L = layout(p.cap);
  double* B = d + L.B;  // B(i, c) = B[i + c * cap]
  double* coup = d + L.coup;
  double* mu = d + L.mu;
  double* nu = d + L.nu;
  double* mun = d + L.mun;
  double* nun = d + L.nun;
  double* sc = d + L.sc;
  const double* res = d + L.res;
  const int t = threadIdx.x;
  const bool alive = iv[I_ALIVE] != 0;
  const int64_t cap = p.cap;
  const int64_t cg_o = R_CG + p.ncols + 3;  // second-pass slots (host cgs2: o = ncols + 3)

  switch (p.op) {
    case OP_L_A:
      run_light(d, iv, p, t, blockDim.x);
      return;
    case OP_L_B:    // after the second pass: omega (left) -> reorthogonalize?
    case OP_R_B: {  // same on the right
      const bool left = p.op == OP_L_B;
      if (!alive) {
        if (t == 0) iv[I_GRE] = iv[I_GRE2] = 0;
        return;
      }
      __shared__ double cand;
      if (t == 0) {
        double c = left ? sc[S_ACAND] : sc[S_BCAND];
        if (iv[I_G2P]) c = sqrt(res[R_N]);
        if (left) sc[S_ACAND] = c; else sc[S_BCAND] = c;
        cand = c;
      }
      __syncthreads();
      extern __shared__ double stg[];
      const bool gre = omega_update(d, p, left, cand, true, stg, t, blockDim.x);
      if (t == 0) {
        iv[I_GRE] = gre ? 1 : 0;
        iv[I_GRE2] = 0;
      }
      return;
    }
    case OP_CG_MID:
      run_light(d, iv, p, t, blockDim.x);
      return;
    case OP_CG_END: {  // cgs2 done: its norm is the new candidate
      const bool on = p.full ? alive : (alive && iv[I_GRE] != 0);
      if (!on) return;
      const bool left = p.side == 0;
      double na = sc[S_NAFTER];
      if (iv[I_GRE2]) na = sqrt(res[cg_o + p.ncols + 1]);
      if (!p.full) {  // partial_reorth_update: committed level after a reorthogonalization
        const int64_t j = p.ncols;
        double* lev = left ? nun : mun;
        for (int64_t i = t; i < j; i += blockDim.x) lev[i] = p.lvl;
      }
      if (t == 0) {
        if (left) sc[S_ACAND] = na; else sc[S_BCAND] = na;
        if (!p.full) iv[I_RPEND] += 1;
      }
      return;
    }
    case OP_SQRT_L: {  // full mode, first step: cgs2 over zero columns = ||w||
      if (alive && t == 0) sc[S_ACAND] = sqrt(res[R_N]);
      return;
    }
    case OP_L_END: {  // alpha fixed: breakdown test, commit column s of B (gkl.cpp:246-262)
      if (!alive) return;
      const int64_t s = p.s;
      const double alpha = sc[S_ACAND];
      const double btol = p.bfac * sc[S_NS];
      if (!(alpha > btol)) {
        if (t == 0) {
          iv[I_STATUS] = 1;
          iv[I_ALIVE] = 0;
        }
        return;
      }
      for (int64_t i = t; i < s; i += blockDim.x) B[i + s * cap] = coup[i];
      for (int64_t i = t; i <= s; i += blockDim.x) nu[i] = p.full ? (i < s ? p.lvl : 1.0) : nun[i];
      if (t == 0) {
        B[s + s * cap] = alpha;
        sc[S_ALPHA] = alpha;
        iv[I_J] = (int)(s + 1);
      }
      return;
    }
    case OP_R_A:
      run_light(d, iv, p, t, blockDim.x);
      return;
    case OP_R_END: {  // beta fixed: breakdown test, coupling, omega levels (gkl.cpp:292-311)
      if (!alive) return;
      const int64_t s = p.s;
      const double beta = sc[S_BCAND];
      const double alpha = sc[S_ALPHA];
      const double btol = p.bfac * sc[S_NS];
      const bool ok = beta > btol;
      __syncthreads();
      for (int64_t i = t; i <= s; i += blockDim.x) coup[i] = 0.0;
      if (ok)
        for (int64_t i = t; i <= s + 1; i += blockDim.x)
          mu[i] = p.full ? (i <= s ? p.lvl : 1.0) : mun[i];
      __syncthreads();
      if (t == 0) {
        iv[I_STEPS] += 1;
        iv[I_REORTH] += iv[I_RPEND];  // svdl counts the reorthogonalizations of completed steps
        iv[I_RPEND] = 0;
        // svdl: norm_scale = max(norm_scale, hypot(alpha, beta)), beta = 0 after
        // a right breakdown (StepInfo.beta is left unset, gkl.cpp:298-300)
        sc[S_NS] = max_ab(sc[S_NS], hypot(alpha, ok ? beta : 0.0));
        if (ok) {
          coup[s] = beta;
          sc[S_BETA] = beta;
        } else {
          iv[I_STATUS] = 2;
          iv[I_ALIVE] = 0;
        }
      }
      return;
    }
    default:
      return;
  }
}

// One decision, or two back to back (then_op >= 0: e.g. the cgs2 end and the
// half-step finalize, consecutive on the critical path) in one launch.
__global__ void __launch_bounds__(kCtlThreads) k_ctl(double* __restrict__ d, int* __restrict__ iv,
                                                     Params p) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  run_op(d, iv, p);
  if (p.then_op >= 0) {
    __syncthreads();  // the first decision's global writes are visible block-wide
    Params q = p;
    q.op = p.then_op;
    q.then_op = -1;
    run_op(d, iv, q);
  }
}

// ---------------------------------------------------------------- fused right tail
// The right half-step after z = X^T u_{s+1} (gkl.cpp:264-311, device-controlled
// as in Lanczos::enqueue_step_dev): (partial mode) z -= alpha v_s with both
// norms -> R_A; the local second pass against v_s (dot, then axpy + norm);
// R_B's omega recurrence; then (gated as cgs2_dev gates it) cgs2 against
// V[:, 0..s] -> CG_MID, second pass, CG_END; R_END. Unfused that is 9 launches
// (5 in full mode), each a kernel boundary on the step's critical path; here
// it is ONE launch of one thread-block cluster for n <= kTailMaxN: the z rows
// stay in registers, each CTA keeps its block partials in shared memory, every
// CTA sums them over DSMEM, and each reduction is one cluster barrier.
//
// Same bits as the unfused kernels (basis_kernels.cu) and k_ctl: virtual block
// b = rows [256 b, 256 b + 256) is reduced exactly as CTA b of those kernels
// reduces it (thread t <-> row 256 b + t, the explicit __fma_rn forms, the
// xor-butterfly warp sums, the eight warp sums in order), the block partials
// are summed in grid_finalize_cols' segment order, and every CTA takes the
// same decisions from the same values (CTA 0 writes them). The dot of the
// second pass is computed with the first reduction (same per-block values as
// k_dot's) and used only when the pass runs; CG_END and R_END are k_ctl's,
// taken on values already in registers.
constexpr int kTT = 256;       // threads (basis_kernels.cu kT: one row per thread per block)
constexpr int kTW = kTT / 32;  // warps = finalize segments (kSeg)
constexpr int kTailR = 4;      // row slots per thread: virtual blocks cta, cta + CL, ...
constexpr int kTCB = 8;        // gemv columns per pass
static_assert(kTailMaxN == 16 * kTT * kTailR, "kernels.hpp kTailMaxN");

__device__ __forceinline__ double wsum(double v) {  // basis_kernels.cu warp_sum
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Eight warp sums at once, reduce-scatter style: at level 16 a lane keeps
// four columns and receives the partner's values of those four (the same
// pair (l, l ^ 16) the plain butterfly adds), then two at level 8, one at 4,
// then a plain butterfly over lanes 2 and 1 -- every column sees the plain
// butterfly's pairings, so the same bits (IEEE addition commutes). Column
// c = (lane >> 2) & 7 ends in lanes 4c..4c+3. 9 shuffles instead of 40.
__device__ __forceinline__ double wsum8(const double (&v)[kTCB]) {
  const int lane = threadIdx.x & 31;
  const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    a[i] = (h4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, h4 ? v[i] : v[i + 4], 16);
#pragma unroll
  for (int i = 0; i < 2; ++i)
    b[i] = (h3 ? a[i + 2] : a[i]) + __shfl_xor_sync(0xffffffffu, h3 ? a[i] : a[i + 2], 8);
  double c = (h2 ? b[1] : b[0]) + __shfl_xor_sync(0xffffffffu, h2 ? b[0] : b[1], 4);
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;
}

// the shared::cluster address of `p` (this CTA's shared memory) in CTA `rank`
__device__ __forceinline__ uint32_t cluster_addr(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  return r;
}

// arrive.release / wait.acquire: the DSMEM partials stored before the barrier
// are visible to every CTA after it
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Combines the per-warp sums ws[m][k][w] of this CTA's slots into block
// partials (eight warp sums in order) in this CTA's spart[vb * K + k0 + k];
// tail_finalize reads them across the cluster.
__device__ void tail_put(int kc, int K, int k0, int cta, int CL, int nblk, double* spart,
                         double (*ws)[kTCB][kTW]) {
  __syncthreads();
  for (int e = threadIdx.x; e < kTailR * kc; e += kTT) {
    const int m = e / kc, k = e - m * kc;
    const int vb = cta + CL * m;
    if (vb >= nblk) continue;
    double tt = 0.0;
#pragma unroll
    for (int w = 0; w < kTW; ++w) tt += ws[m][k][w];
    spart[(int64_t)vb * K + k0 + k] = tt;
  }
  __syncthreads();  // ws reusable
}

// Block partials of K <= kTCB columns: v[k][m] is the thread's value for
// column k in slot m.
template <int K>
__device__ void tail_partials(const double (&v)[K][kTailR], int cta, int CL, int nblk,
                              double* spart, double (*ws)[kTCB][kTW]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < kTailR; ++m) {
    if (cta + CL * m >= nblk) break;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double w = wsum(v[k][m]);
      if (lane == 0) ws[m][k][warp] = w;
    }
  }
  tail_put(K, K, 0, cta, CL, nblk, spart, ws);
}

// grid_finalize_cols' sums of columns [0, K) over the nblk partials (block
// vb's in CTA vb % CL), into fin[]; a warp's segment loads are independent.
__device__ void tail_finalize(const double* spart, int nblk, int K, double* fin,
                              double (*seg)[33]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, CL = (int)gridDim.x;
  const int b0 = (int)((int64_t)nblk * warp / kTW), b1 = (int)((int64_t)nblk * (warp + 1) / kTW);
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int k = k0 + lane;
    double t = 0.0;
    if (k < K) {
      // all of the segment's loads issued, then summed in order
      constexpr int kMaxSeg = (16 * kTailR + kTW - 1) / kTW;
      double v[kMaxSeg];
#pragma unroll
      for (int i = 0; i < kMaxSeg; ++i)
        if (b0 + i < b1)
          asm volatile("ld.shared::cluster.f64 %0, [%1];"
                       : "=d"(v[i])
                       : "r"(cluster_addr(spart + (int64_t)(b0 + i) * K + k, (b0 + i) % CL))
                       : "memory");
#pragma unroll
      for (int i = 0; i < kMaxSeg; ++i)
        if (b0 + i < b1) t += v[i];
    }
    seg[warp][lane] = t;
    __syncthreads();
    if (warp == 0 && k < K) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kTW; ++w) s += seg[w][lane];
      fin[k] = s;
    }
    __syncthreads();
  }
}

// gemv_t (k_gemv_t) over this CTA's rows: partials of Q[:, c]^T z for
// c < ncols, ||z||^2 at c = ncols when K = ncols + 1. Every slot's loads of a
// column group are issued together.
__device__ __forceinline__ void tail_load8(const double* __restrict__ Q, int64_t n, int64_t ncols,
                                           int c0, const int64_t (&rows)[kTailR],
                                           double (&q)[kTailR][kTCB]) {
#pragma unroll
  for (int m = 0; m < kTailR; ++m)
#pragma unroll
    for (int k = 0; k < kTCB; ++k) {
      const int64_t c = c0 + k;
      q[m][k] = (c < ncols && rows[m] >= 0) ? Q[c * n + rows[m]] : 0.0;
    }
}

__device__ void tail_gemv_t(const double* __restrict__ Q, int64_t n, int64_t ncols, int K,
                            const double (&zr)[kTailR], int cta, int CL, int nblk, double* spart,
                            double (*ws)[kTCB][kTW]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t rows[kTailR];
#pragma unroll
  for (int m = 0; m < kTailR; ++m) {
    const int64_t row = (int64_t)(cta + CL * m) * kTT + t;
    rows[m] = (cta + CL * m < nblk && row < n) ? row : -1;
  }
  for (int c0 = 0; c0 < K; c0 += kTCB) {
    double q[kTailR][kTCB];
    tail_load8(Q, n, ncols, c0, rows, q);
#pragma unroll
    for (int m = 0; m < kTailR; ++m) {
      if (cta + CL * m >= nblk) break;
      double vals[kTCB];
#pragma unroll
      for (int k = 0; k < kTCB; ++k) {
        const int64_t c = c0 + k;
        vals[k] = c < ncols ? __fma_rn(q[m][k], zr[m], 0.0)
                            : (c == ncols && c < K ? __fma_rn(zr[m], zr[m], 0.0) : 0.0);
      }
      const double w = wsum8(vals);
      if ((lane & 3) == 0) ws[m][lane >> 2][warp] = w;
    }
    tail_put(min(kTCB, K - c0), K, c0, cta, CL, nblk, spart, ws);
  }
}

// gemv_n (k_gemv_n, beta 1, sign -1): z -= Q c over this CTA's rows, with the
// norms before / after as two block-partial columns.
__device__ void tail_gemv_n(const double* __restrict__ Q, int64_t n, int64_t ncols,
                            const double* __restrict__ cf, double (&zr)[kTailR], int cta, int CL,
                            int nblk, double* spart, double (*ws)[kTCB][kTW]) {
  const int t = threadIdx.x;
  double acc[kTailR];
  int64_t rows[kTailR];
#pragma unroll
  for (int m = 0; m < kTailR; ++m) {
    acc[m] = 0.0;
    const int64_t row = (int64_t)(cta + CL * m) * kTT + t;
    rows[m] = (cta + CL * m < nblk && row < n) ? row : -1;
  }
  // column groups of kTCB, every slot's loads of a group in flight together
  for (int64_t l = 0; l < ncols; l += kTCB) {
    double q[kTailR][kTCB];
    tail_load8(Q, n, ncols, (int)l, rows, q);
#pragma unroll
    for (int m = 0; m < kTailR; ++m)
#pragma unroll
      for (int k = 0; k < kTCB; ++k)
        if (l + k < ncols) acc[m] = __fma_rn(q[m][k], cf[l + k], acc[m]);
  }
  double nr[2][kTailR];
#pragma unroll
  for (int m = 0; m < kTailR; ++m) {
    nr[0][m] = nr[1][m] = 0.0;
    if (rows[m] < 0) continue;
    const double old = zr[m];
    const double nv = __fma_rn(1.0, old, __dmul_rn(-1.0, acc[m]));
    zr[m] = nv;
    nr[0][m] = __fma_rn(old, old, 0.0);
    nr[1][m] = __fma_rn(nv, nv, 0.0);
  }
  tail_partials<2>(nr, cta, CL, nblk, spart, ws);
}

// GKB_RTAIL_TLOG: CTA 0 accumulates the cycles of each phase (debug timeline;
// slot 15 counts launches)
struct TailClock {
  unsigned long long* log;
  long long t0;
  __device__ void mark(int slot) {
    if (!log || blockIdx.x != 0 || threadIdx.x != 0) return;
    const long long t = clock64();
    atomicAdd(log + slot, (unsigned long long)(t - t0));
    t0 = t;
  }
};

__global__ void __launch_bounds__(kTT) k_right_tail(TailArgs a) {
  pdl_wait();  // (pdl.hpp) nothing before this reads or writes global memory
  pdl_trigger();
  TailClock clk{a.tlog, clock64()};
  if (a.tlog && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.tlog + 15, 1ull);
  // dynamic smem: kStageBytes omega staging | fin[cap + 8] | two partial buffers
  extern __shared__ double dsm[];
  const Params& p = a.p;
  const int64_t n = a.n, s = p.s, ncols = s + 1;
  const int nblk = (int)((n + kTT - 1) / kTT);
  double* stg = dsm;
  double* fin = dsm + kStageBytes / sizeof(double);
  double* spart[2] = {fin + p.cap + 8, fin + p.cap + 8 + (int64_t)nblk * (ncols + 1)};
  __shared__ double ws[kTailR][kTCB][kTW];
  __shared__ double seg[kTW][33];
  const Layout L = layout(p.cap);
  double* d = a.d;
  int* iv = a.iv;
  double* sc = d + L.sc;
  double* res = d + L.res;
  const int t = threadIdx.x, CL = (int)gridDim.x, cta = (int)blockIdx.x;
  const bool w0 = cta == 0 && t == 0;  // the scalar writer
  const bool full = p.full != 0;
  // every scalar the tail reads, in one round trip with the z rows
  const bool alive = iv[I_ALIVE] != 0;
  const double alpha = sc[S_ALPHA], ns = sc[S_NS];
  int steps = 0, reorth = 0, rpend = 0;
  if (w0) {
    steps = iv[I_STEPS];
    reorth = iv[I_REORTH];
    rpend = iv[I_RPEND];
  }
  double zr[kTailR], vr[kTailR];
#pragma unroll
  for (int m = 0; m < kTailR; ++m) {
    const int64_t row = (int64_t)(cta + CL * m) * kTT + t;
    const bool ok = cta + CL * m < nblk && row < n;
    zr[m] = ok ? a.z[row] : 0.0;
    vr[m] = (!full && ok) ? a.V[s * n + row] : 0.0;
  }
  if (!alive) {  // every gated kernel off; the decisions' dead branches
    if (w0) {
      if (!full) iv[I_G2P] = iv[I_GRE] = 0;
      iv[I_GRE2] = 0;
    }
    return;
  }
  clk.mark(0);  // scalars, z and v_s rows loaded
  int ph = 0;
  bool gre = full;
  double cand = 0.0, est = 0.0;
  if (!full) {
    // axpy_norms_dv + R_A: z -= alpha v_s, ||z||^2 before / after; with them
    // v_s . z (k_dot's block values), used if the local second pass runs
    double v3[3][kTailR];
#pragma unroll
    for (int m = 0; m < kTailR; ++m) {
      const double x = zr[m];
      const double nv = __fma_rn(-alpha, vr[m], x);
      v3[0][m] = __fma_rn(x, x, 0.0);
      v3[1][m] = __fma_rn(nv, nv, 0.0);
      v3[2][m] = __fma_rn(vr[m], nv, 0.0);
      zr[m] = nv;
    }
    tail_partials<3>(v3, cta, CL, nblk, spart[ph], ws);
    clk.mark(1);  // block partials stored
    cluster_sync_all();
    clk.mark(2);  // cluster barrier
    tail_finalize(spart[ph], nblk, 3, fin, seg);
    clk.mark(3);  // finalize
    ph ^= 1;
    const double n0 = fin[0], n1 = fin[1], dv = fin[2];
    const double bc = sqrt(n1);
    const bool g2p = bc < p.eta * sqrt(n0);
    if (w0) {
      res[R_N] = n0;
      res[R_N + 1] = n1;
      iv[I_G2P] = g2p ? 1 : 0;
    }
    cand = bc;
    if (g2p) {  // local second pass against v_s (gkl.cpp:277-284): axpy + norm
      if (w0) res[R_DOT] = dv;
      double v1[1][kTailR];
#pragma unroll
      for (int m = 0; m < kTailR; ++m) {
        zr[m] = __fma_rn(-dv, vr[m], zr[m]);
        v1[0][m] = __fma_rn(zr[m], zr[m], 0.0);
      }
      tail_partials<1>(v1, cta, CL, nblk, spart[ph], ws);
      cluster_sync_all();
      tail_finalize(spart[ph], nblk, 1, fin, seg);
      ph ^= 1;
      if (w0) res[R_N] = fin[0];
      cand = sqrt(fin[0]);
    }
    clk.mark(4);  // local second pass
    // R_B: the omega recurrence -> reorthogonalize? (every CTA; levels kept
    // in registers, committed with R_END)
    gre = omega_update(d, p, false, cand, false, stg, t, kTT, &est);
    if (w0) {
      iv[I_GRE] = gre ? 1 : 0;
      iv[I_GRE2] = 0;
    }
    clk.mark(5);  // omega recurrence
  }
  double bfin = cand;  // the beta candidate R_END tests
  if (gre) {  // cgs2 against V[:, 0..s] (orth.hpp:19-44), as cgs2_dev
    tail_gemv_t(a.V, n, ncols, (int)ncols + 1, zr, cta, CL, nblk, spart[ph], ws);
    clk.mark(6);  // gemv_t partials
    cluster_sync_all();
    clk.mark(7);  // cluster barrier
    tail_finalize(spart[ph], nblk, (int)ncols + 1, fin, seg);
    clk.mark(9);  // finalize
    ph ^= 1;
    if (cta == 0)
      for (int64_t k = t; k <= ncols; k += kTT) res[R_CG + k] = fin[k];
    const double nb = sqrt(fin[ncols]);
    tail_gemv_n(a.V, n, ncols, fin, zr, cta, CL, nblk, spart[ph], ws);
    clk.mark(10);  // gemv_n
    cluster_sync_all();
    tail_finalize(spart[ph], nblk, 2, fin, seg);
    clk.mark(11);  // cluster barrier + finalize
    ph ^= 1;
    const double na = sqrt(fin[1]);
    const bool gre2 = na < p.eta * nb;  // CG_MID
    if (w0) {
      res[R_CG + ncols + 1] = fin[0];
      res[R_CG + ncols + 2] = fin[1];
      iv[I_GRE2] = gre2 ? 1 : 0;
      sc[S_NAFTER] = na;
    }
    bfin = na;
    if (gre2) {
      const int64_t o2 = R_CG + ncols + 3;
      tail_gemv_t(a.V, n, ncols, (int)ncols, zr, cta, CL, nblk, spart[ph], ws);
      cluster_sync_all();
      tail_finalize(spart[ph], nblk, (int)ncols, fin, seg);
      ph ^= 1;
      if (cta == 0)
        for (int64_t k = t; k < ncols; k += kTT) res[o2 + k] = fin[k];
      tail_gemv_n(a.V, n, ncols, fin, zr, cta, CL, nblk, spart[ph], ws);
      cluster_sync_all();
      tail_finalize(spart[ph], nblk, 2, fin, seg);
      ph ^= 1;
      if (w0) {
        res[o2 + ncols] = fin[0];
        res[o2 + ncols + 1] = fin[1];
      }
      bfin = sqrt(fin[1]);  // CG_END: the second pass's norm
      clk.mark(12);  // second pass
      if (a.tlog && w0) atomicAdd(a.tlog + 14, 1ull);
    }
  } else if (w0) {
    iv[I_GRE2] = 0;  // CG_MID of a gated-off cgs2
  }
  if (a.tlog && w0) {
    if (gre) atomicAdd(a.tlog + 13, 1ull);
  }
#pragma unroll
  for (int m = 0; m < kTailR; ++m) {
    const int64_t row = (int64_t)(cta + CL * m) * kTT + t;
    if (cta + CL * m < nblk && row < n) a.z[row] = zr[m];
  }
  if (cta != 0) return;
  // CG_END + R_END (k_ctl run_op) on register values: the levels (mun: the
  // recurrence's estimates, or lvl after a reorthogonalization), the beta
  // candidate, the counters
  const bool ok = bfin > p.bfac * ns;
  const int64_t j = ncols;
  double* coup = d + L.coup;
  double* mu = d + L.mu;
  double* mun = d + L.mun;
  for (int64_t i = t; i <= s + 1; i += kTT) {
    double lev = 1.0;  // mun[j]
    if (!full) {
      if (i < j) lev = gre ? p.lvl : est;
      mun[i] = lev;
    }
    if (i <= s) coup[i] = (i == s && ok) ? bfin : 0.0;
    if (ok) mu[i] = full ? (i <= s ? p.lvl : 1.0) : lev;
  }
  if (t == 0) {
    iv[I_RPEND] = 0;
    iv[I_REORTH] = reorth + rpend + ((!full && gre) ? 1 : 0);
    iv[I_STEPS] = steps + 1;
    sc[S_BCAND] = bfin;
    sc[S_NS] = max_ab(ns, hypot(alpha, ok ? bfin : 0.0));
    if (ok) {
      sc[S_BETA] = bfin;
    } else {
      iv[I_STATUS] = 2;
      iv[I_ALIVE] = 0;
    }
  }
  clk.mark(8);  // CG_END + R_END
}

}  // namespace

void launch(double* d, int* iv, const Params& p, cudaStream_t st) {
  launch_pdl(k_ctl, dim3(1), dim3(kCtlThreads), kStageBytes, st, true, d, iv, p);
}


// One cluster of min(16, blocks) CTAs; false (nothing launched) when the
// fused tail does not apply: n > kTailMaxN, a basis wider than the level
// staging, GKB_NO_RTAIL set, or no cluster launch.
bool right_tail(const TailArgs& a, cudaStream_t st) {
  const bool off = getenv("GKB_NO_RTAIL") != nullptr || getenv("GKB_GT_BLOCKS") != nullptr ||
                   getenv("GKB_GN_BLOCKS") != nullptr;
  // partial mode only: in full mode the tail is two cgs2 passes over V, which
  // one cluster streams slower than the full-grid kernels (config 1: +1.5%)
  if (off || a.p.full || a.n <= 0 || a.n > kTailMaxN) return false;
  const int64_t nblk = (a.n + kTT - 1) / kTT;
  const int64_t ncols = a.p.s + 1;
  if (ncols > kStageJ) return false;
  const int CL = (int)std::min<int64_t>(16, nblk);
  if (nblk > (int64_t)CL * kTailR) return false;
  const size_t smem =
      kStageBytes + sizeof(double) * (size_t)(a.p.cap + 8 + 2 * nblk * (ncols + 1));
  static int ready = 0;  // 1: attributes set, -1: unsupported
  if (ready == 0) {
    ready = (cudaFuncSetAttribute(k_right_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                 cudaSuccess &&
             cudaFuncSetAttribute(k_right_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  160 * 1024) == cudaSuccess)
                ? 1
                : -1;
    if (ready < 0) cudaGetLastError();
  }
  if (ready < 0 || smem > 160 * 1024) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)CL);
  cfg.blockDim = dim3(kTT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_right_tail, a);
  if (e != cudaSuccess) {
    cudaGetLastError();
    static bool told = false;
    if (!told) fprintf(stderr, "[gkb] fused right tail not launched (%s): unfused path\n",
                       cudaGetErrorString(e));
    told = true;
    ready = -1;
    return false;
  }
  return true;
}

}  // namespace ctl
}  // namespace dev
}  // namespace gkb
