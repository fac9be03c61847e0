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
