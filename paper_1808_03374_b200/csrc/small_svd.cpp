// svd_small (small_svd.cpp:14-28 of the reference): the projected problem
// stays on the host (BASELINE north star item 3). SPEC.md's design decision
// names one-sided Jacobi "for accuracy on small projected matrices"; this is
// Hestenes' cyclic method with accumulated right rotations, singular values
// sorted descending, and an orthonormal completion for numerically null
// directions so both factors always have orthonormal columns.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <numeric>
#include <vector>

#include "host.hpp"

namespace gkb {

namespace {

// x.y with four interleaved partial sums (short dependency chains; fixed order)
inline double dot4(const double* x, const double* y, int64_t r) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t i = 0;
  for (; i + 4 <= r; i += 4) {
    s0 += x[i] * y[i];
    s1 += x[i + 1] * y[i + 1];
    s2 += x[i + 2] * y[i + 2];
    s3 += x[i + 3] * y[i + 3];
  }
  for (; i < r; ++i) s0 += x[i] * y[i];
  return (s0 + s1) + (s2 + s3);
}

// A (r x c, r >= c) -> U (r x c), s (c), V (c x c). An AVX2 clone where the
// host has it: the loops vectorize lane-for-lane (dot4's four sums are the
// four lanes, no FMA contraction), so both clones give the same bits. (A
// round-robin ordering with the rounds shared among OpenMP threads was slower:
// ~100 rounds per sweep of ~25 pairs at ~50 ns each do not pay two barriers.)
__attribute__((target_clones("avx2", "default")))
void jacobi_tall(const double* M, int64_t r, int64_t c, double* U, double* s, double* V) {
  std::vector<double> A(M, M + r * c), R((size_t)(c * c), 0.0);
  for (int64_t i = 0; i < c; ++i) R[i + i * c] = 1.0;
  // column norms: recomputed at the start of every sweep, updated exactly as
  // the rotation changes them in between (a_p.a_p - t g, a_q.a_q + t g)
  std::vector<double> nrm((size_t)c);
  for (int sweep = 0; sweep < 80; ++sweep) {
    for (int64_t p = 0; p < c; ++p) {
      const double* ap = A.data() + p * r;
      nrm[p] = dot4(ap, ap, r);
    }
    bool rotated = false;
    for (int64_t p = 0; p + 1 < c; ++p) {
      double* ap = A.data() + p * r;
      for (int64_t q = p + 1; q < c; ++q) {
        double* aq = A.data() + q * r;
        const double gamma = dot4(ap, aq, r);
        const double alpha = nrm[p], beta = nrm[q];
        if (gamma == 0.0 || std::fabs(gamma) <= DBL_EPSILON * std::sqrt(alpha) * std::sqrt(beta))
          continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::hypot(1.0, zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int64_t i = 0; i < r; ++i) {
          const double x = ap[i], y = aq[i];
          ap[i] = cs * x - sn * y;
          aq[i] = sn * x + cs * y;
        }
        nrm[p] = alpha - t * gamma;
        nrm[q] = beta + t * gamma;
        double* rp = R.data() + p * c;
        double* rq = R.data() + q * c;
        for (int64_t i = 0; i < c; ++i) {
          const double x = rp[i], y = rq[i];
          rp[i] = cs * x - sn * y;
          rq[i] = sn * x + cs * y;
        }
      }
    }
    if (!rotated) break;
  }
  std::vector<double> sv((size_t)c);
  for (int64_t i = 0; i < c; ++i) {
    double t = 0.0;
    for (int64_t k = 0; k < r; ++k) t += A[i * r + k] * A[i * r + k];
    sv[i] = std::sqrt(t);
  }
  std::vector<int64_t> order((size_t)c);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return sv[a] > sv[b]; });
  const double smax = c > 0 ? sv[order[0]] : 0.0;
  const double zero_tol = smax * DBL_EPSILON * (double)std::max(r, c);
  for (int64_t i = 0; i < c; ++i) {
    const int64_t src = order[i];
    s[i] = sv[src];
    std::copy(R.begin() + src * c, R.begin() + (src + 1) * c, V + i * c);
    double* u = U + i * r;
    if (sv[src] > zero_tol && sv[src] > 0.0) {
      for (int64_t k = 0; k < r; ++k) u[k] = A[src * r + k] / sv[src];
      continue;
    }
    for (int64_t e = 0; e < r; ++e) {
      for (int64_t k = 0; k < r; ++k) u[k] = (k == e) ? 1.0 : 0.0;
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t l = 0; l < i; ++l) {
          const double* ul = U + l * r;
          double d = 0.0;
          for (int64_t k = 0; k < r; ++k) d += ul[k] * u[k];
          for (int64_t k = 0; k < r; ++k) u[k] -= d * ul[k];
        }
      double nn = 0.0;
      for (int64_t k = 0; k < r; ++k) nn += u[k] * u[k];
      nn = std::sqrt(nn);
      if (nn > 0.5) {
        for (int64_t k = 0; k < r; ++k) u[k] /= nn;
        break;
      }
    }
  }
}

}  // namespace

void svd_small(const double* M, int64_t r, int64_t c, double* U, double* s, double* V) {
  if (r <= 0 || c <= 0) return;
  if (r >= c) {
    jacobi_tall(M, r, c, U, s, V);
    return;
  }
  std::vector<double> T((size_t)(r * c));
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < c; ++j) T[j + i * c] = M[i + j * r];
  jacobi_tall(T.data(), c, r, V, s, U);
}

}  // namespace gkb
