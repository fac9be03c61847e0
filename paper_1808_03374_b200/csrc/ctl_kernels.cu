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

#include <cstdint>

#include "kernels.hpp"
#include "pdl.hpp"
#include "ctl_ops.cuh"

namespace gkb {
namespace dev {
namespace ctl {

namespace {

constexpr int kCtlThreads = 128;
constexpr int64_t kStageJ = 64;  // factorizations up to this size staged in shared memory
constexpr size_t kStageBytes = sizeof(double) * (size_t)(kStageJ * kStageJ + 3 * (kStageJ + 2));

// std::min(1.0, x) / std::max(a, b) exactly as <algorithm> defines them
__device__ __forceinline__ double min_1(double x) { return (x < 1.0) ? x : 1.0; }
__device__ __forceinline__ double max_ab(double a, double b) { return (a < b) ? b : a; }

// max over the CTA of per-thread maxima (each started at 0.0 and folded with
// max_ab; NaN estimates never enter, as in the host loop). Max is exact, so
// the grouping does not matter.
__device__ double block_max(double v) {
  __shared__ double sm[kCtlThreads / 32];
  for (int o = 16; o > 0; o >>= 1) v = max_ab(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  double w = 0.0;
  for (int i = 0; i < kCtlThreads / 32; ++i) w = max_ab(w, sm[i]);
  __syncthreads();
  return w;
}

__device__ bool monitors_side(bool left, const Params& p, double norm_scale) {
  if (!p.one_sided || norm_scale > p.guard) return true;  // gkl.cpp:27-33
  return left ? p.m <= p.n : p.n < p.m;
}

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
  const double tau = 2.0 * p.lvl * sc[S_NS] + p.lvl;
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
      const int64_t j = left ? p.s : p.s + 1;  // factorization size at this half-step
      // The recurrences read the leading j x j block of B and the level rows:
      // staged in shared memory (one coalesced pass) when they fit, so the
      // per-i sequential sums below run at shared-memory latency.
      extern __shared__ double stg[];
      const bool staged = j <= kStageJ;
      const double* Bs = B;
      int64_t lds = cap;
      const double *mus = mu, *nus = nu, *cps = coup;
      if (staged) {
        double* sB = stg;
        double* smu = sB + kStageJ * kStageJ;
        double* snu = smu + kStageJ + 2;
        double* scp = snu + kStageJ + 2;
        // warp w copies columns w, w + 4, ...; lanes the rows (no 64-bit div/mod)
        const int jj = (int)j, lane = t & 31, nw = (int)(blockDim.x >> 5);
        for (int c = t >> 5; c < jj; c += nw)
          for (int i = lane; i < jj; i += 32) sB[i + c * jj] = B[i + (int64_t)c * cap];
        for (int64_t e = t; e <= j; e += blockDim.x) {
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
      const double denom = max_ab(cand, tau + p.eps);
      double worst = 0.0;
      if (left) {
        for (int64_t i = t; i < j; i += blockDim.x) {
          double acc = 0.0;
          for (int64_t c = i; c < j; ++c) acc += fabs(Bs[i + c * lds]) * mus[c];
          if (p.omega_rec == 1)
            for (int64_t c = 0; c < j; ++c)
              if (c != i && cps[c] != 0.0) acc += fabs(cps[c]) * nus[c < i ? c : i];
          const double est = min_1((acc + tau) / denom);
          nun[i] = est;
          worst = max_ab(worst, est);
        }
        if (t == 0) nun[j] = 1.0;
      } else {
        const double alpha_last = Bs[(j - 1) + (j - 1) * lds];
        for (int64_t i = t; i < j; i += blockDim.x) {
          double acc = 0.0;
          if (i == j - 1) {
            for (int64_t r = 0; r + 1 < j; ++r) acc += fabs(Bs[r + i * lds]) * nus[r];
          } else {
            for (int64_t r = 0; r <= i; ++r) acc += fabs(Bs[r + i * lds]) * nus[r];
            acc += alpha_last * mus[i];
          }
          const double est = min_1((acc + tau) / denom);
          mun[i] = est;
          worst = max_ab(worst, est);
        }
        if (t == 0) mun[j] = 1.0;
      }
      worst = block_max(worst);
      if (t == 0) {
        iv[I_GRE] = (worst > p.omega && monitors_side(left, p, sc[S_NS])) ? 1 : 0;
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

}  // namespace

void launch(double* d, int* iv, const Params& p, cudaStream_t st) {
  launch_pdl(k_ctl, dim3(1), dim3(kCtlThreads), kStageBytes, st, true, d, iv, p);
}

}  // namespace ctl
}  // namespace dev
}  // namespace gkb
