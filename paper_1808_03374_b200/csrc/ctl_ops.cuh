// Light step-control decisions (ctl_kernels.cu) shared with the
// reduction kernels: L_A (local second pass on the left?), R_A (on the
// right?), CG_MID (cgs2 second pass?). They only take square roots and compare
// products (no a*b+c to contract), so they give the same bits in either file.
// Run by one CTA: thread t of nt.
#pragma once

#include "kernels.hpp"

namespace gkb {
namespace dev {
namespace ctl {

__device__ inline bool light_op(int op) { return op == OP_L_A || op == OP_R_A || op == OP_CG_MID; }

// std::min(1.0, x) / std::max(a, b) exactly as <algorithm> defines them
__device__ __forceinline__ double min_1(double x) { return (x < 1.0) ? x : 1.0; }
__device__ __forceinline__ double max_ab(double a, double b) { return (a < b) ? b : a; }

// max over the CTA (nt threads, a multiple of 32, <= 1024) of per-thread
// maxima (each started at 0.0 and folded with max_ab; NaN estimates never
// enter, as in the host loop). Max is exact, so the grouping does not matter.
__device__ inline double block_max(double v, int nt) {
  __shared__ double bm_sm[32];
  for (int o = 16; o > 0; o >>= 1) v = max_ab(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) bm_sm[threadIdx.x >> 5] = v;
  __syncthreads();
  double w = 0.0;
  for (int i = 0; i < nt / 32; ++i) w = max_ab(w, bm_sm[i]);
  __syncthreads();
  return w;
}

__device__ inline bool monitors_side(bool left, const Params& p, double norm_scale) {
  if (!p.one_sided || norm_scale > p.guard) return true;  // gkl.cpp:27-33
  return left ? p.m <= p.n : p.n < p.m;
}

constexpr int64_t kStageJ = 64;  // factorizations up to this size staged in shared memory
constexpr size_t kStageBytes = sizeof(double) * (size_t)(kStageJ * kStageJ + 3 * (kStageJ + 2));

// OP_L_B / OP_R_B after the candidate norm `cand` is known: the omega
// recurrence of partial_reorth_update (gkl.cpp:112-176) for the side, and the
// reorthogonalize decision, returned to every thread. `wr`: commit the new
// level row (nun / mun) -- the fused right tail (basis_kernels.cu) runs this in
// every CTA of its cluster and lets one write. The products and sums are
// explicit __dmul_rn / __dadd_rn: the same bits whether the including file is
// compiled with FMA contraction (basis_kernels.cu) or without (ctl_kernels.cu,
// matching the host's -ffp-contract=off). `stg`: kStageBytes of dynamic smem.
// `my_est`: the thread's level estimate for row i = t (when j <= nt).
__device__ inline bool omega_update(double* __restrict__ d, const Params& p, bool left, double cand,
                                    bool wr, double* stg, int t, int nt, double* my_est = nullptr) {
  const Layout L = layout(p.cap);
  const double* B = d + L.B;  // B(i, c) = B[i + c * cap]
  const double* coup = d + L.coup;
  const double* mu = d + L.mu;
  const double* nu = d + L.nu;
  double* mun = d + L.mun;
  double* nun = d + L.nun;
  const double* sc = d + L.sc;
  const int64_t cap = p.cap;
  const double tau = __dadd_rn(__dmul_rn(__dmul_rn(2.0, p.lvl), sc[S_NS]), p.lvl);
  const int64_t j = left ? p.s : p.s + 1;  // factorization size at this half-step
  // The recurrences read the leading j x j block of B and the level rows:
  // staged in shared memory (one coalesced pass) when they fit, so the
  // per-i sequential sums below run at shared-memory latency.
  const bool staged = j <= kStageJ;
  const double* Bs = B;
  int64_t lds = cap;
  const double *mus = mu, *nus = nu, *cps = coup;
  if (staged) {
    double* sB = stg;
    double* smu = sB + kStageJ * kStageJ;
    double* snu = smu + kStageJ + 2;
    double* scp = snu + kStageJ + 2;
    // batches of 16 loads per thread issued before their stores (one L2
    // round trip per batch, not one per column): element e = i + c jj
    const int jj = (int)j, nel = jj * jj;
    for (int base = 0; base < nel; base += 16 * nt) {
      double tmp[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int e = base + t + k * nt;
        if (e < nel) {
          const int c = e / jj;
          tmp[k] = B[(e - c * jj) + (int64_t)c * cap];
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int e = base + t + k * nt;
        if (e < nel) sB[e] = tmp[k];
      }
    }
    for (int64_t e = t; e <= j; e += nt) {
      smu[e] = mu[e];
      snu[e] = nu[e];
      scp[e] = e < cap ? coup[e] : 0.0;
    }
    Bs = sB;
    lds = j;
    mus = smu;
    nus = snu;
    cps = scp;
  }
  __syncthreads();
  const double denom = max_ab(cand, __dadd_rn(tau, p.eps));
  double worst = 0.0;
  if (left) {
    for (int64_t i = t; i < j; i += nt) {
      double acc = 0.0;
      for (int64_t c = i; c < j; ++c) acc = __dadd_rn(acc, __dmul_rn(fabs(Bs[i + c * lds]), mus[c]));
      if (p.omega_rec == 1)
        for (int64_t c = 0; c < j; ++c)
          if (c != i && cps[c] != 0.0)
            acc = __dadd_rn(acc, __dmul_rn(fabs(cps[c]), nus[c < i ? c : i]));
      const double est = min_1(__ddiv_rn(__dadd_rn(acc, tau), denom));
      if (wr) nun[i] = est;
      if (my_est && i == t) *my_est = est;
      worst = max_ab(worst, est);
    }
    if (wr && t == 0) nun[j] = 1.0;
  } else {
    const double alpha_last = Bs[(j - 1) + (j - 1) * lds];
    for (int64_t i = t; i < j; i += nt) {
      double acc = 0.0;
      if (i == j - 1) {
        for (int64_t r = 0; r + 1 < j; ++r) acc = __dadd_rn(acc, __dmul_rn(fabs(Bs[r + i * lds]), nus[r]));
      } else {
        for (int64_t r = 0; r <= i; ++r) acc = __dadd_rn(acc, __dmul_rn(fabs(Bs[r + i * lds]), nus[r]));
        acc = __dadd_rn(acc, __dmul_rn(alpha_last, mus[i]));
      }
      const double est = min_1(__ddiv_rn(__dadd_rn(acc, tau), denom));
      if (wr) mun[i] = est;
      if (my_est && i == t) *my_est = est;
      worst = max_ab(worst, est);
    }
    if (wr && t == 0) mun[j] = 1.0;
  }
  worst = block_max(worst, nt);
  return worst > p.omega && monitors_side(left, p, sc[S_NS]);
}

__device__ inline void run_light(double* __restrict__ d, int* __restrict__ iv, const Params& p,
                                 int t, int nt) {
  const Layout L = layout(p.cap);
  const double* coup = d + L.coup;
  double* sc = d + L.sc;
  const double* res = d + L.res;
  const bool alive = iv[I_ALIVE] != 0;
  const int64_t cap = p.cap;
  switch (p.op) {
    case OP_L_A: {  // norms of the left candidate -> local second pass?
      if (!alive) {
        if (t == 0) iv[I_G2P] = iv[I_GRE] = iv[I_GRE2] = 0;
        for (int64_t c = t; c < cap; c += nt) iv[I_G2PC + c] = 0;
        return;
      }
      const double w0 = sqrt(res[R_N]);
      const double ac = sqrt(res[R_N + p.nidx]);
      const bool f = ac < p.eta * w0;
      for (int64_t c = t; c < cap; c += nt)
        iv[I_G2PC + c] = (f && p.has_pattern && c >= p.lo && c <= p.hi && coup[c] != 0.0) ? 1 : 0;
      if (t == 0) {
        iv[I_G2P] = (f && p.has_pattern) ? 1 : 0;
        sc[S_ACAND] = ac;
      }
      return;
    }
    case OP_CG_MID: {  // cgs2 pass 1 done: second pass? (orth.hpp:30-33)
      const bool on = p.full ? alive : (alive && iv[I_GRE] != 0);
      if (t != 0) return;
      if (!on) {
        iv[I_GRE2] = 0;
        return;
      }
      const double nb = sqrt(res[R_CG + p.ncols]);
      const double na = sqrt(res[R_CG + p.ncols + 2]);
      iv[I_GRE2] = (na < p.eta * nb) ? 1 : 0;
      sc[S_NAFTER] = na;
      return;
    }
    case OP_R_A: {  // norms of the right candidate -> local second pass? (partial)
      if (!alive) {
        if (t == 0) iv[I_G2P] = iv[I_GRE] = iv[I_GRE2] = 0;
        return;
      }
      if (t == 0) {
        const double z0 = sqrt(res[R_N]);
        const double bc = sqrt(res[R_N + 1]);
        iv[I_G2P] = (bc < p.eta * z0) ? 1 : 0;
        sc[S_BCAND] = bc;
      }
      return;
    }
    default:
      return;
  }
}

}  // namespace ctl
}  // namespace dev
}  // namespace gkb
