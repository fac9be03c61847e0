/*
 * gkb_oracle.c -- CPU restatement of the reference GKL hot path.
 * TEST INFRASTRUCTURE ONLY (see gkb_oracle.h): the checker and the CPU
 * baseline, never linked into the product library.
 *
 * Compiled with -ffp-contract=off so that every floating-point expression is
 * evaluated exactly as written (no fused multiply-add); the marker scaling
 * formula must reproduce the product's host code bit for bit.
 */
#include "gkb_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_EPS DBL_EPSILON

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) {
    fprintf(stderr, "gkb_oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ======================================================================
 * Rng -- rng.hpp:17-62. The engine is std::mt19937_64 (seeded with
 * the 64-bit Knuth initializer, i.e. std::mersenne_twister_engine's
 * seed(value) algorithm); draws follow rng.hpp exactly.
 * ==================================================================== */
#define MT_NN 312
#define MT_MM 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_init(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_NN;
  r->spare = 0.0;
  r->have_spare = 0;
}

uint64_t orc_rng_bits(orc_rng* r) {
  if (r->mti >= MT_NN) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
      r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
    }
    for (; i < MT_NN - 1; ++i) {
      x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
      r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
    }
    x = (r->mt[MT_NN - 1] & MT_UM) | (r->mt[0] & MT_LM);
    r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:24 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_bits(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:27 */
double orc_rng_uniform_symmetric(orc_rng* r) { return 2.0 * orc_rng_uniform(r) - 1.0; }

/* rng.hpp:30-38 */
uint64_t orc_rng_uniform_int(orc_rng* r, uint64_t lo, uint64_t hi) {
  if (lo > hi) return lo; /* reference throws; callers never do this */
  const uint64_t span = hi - lo + 1;
  if (span == 0) return orc_rng_bits(r);
  const uint64_t reject_above = UINT64_MAX - UINT64_MAX % span;
  uint64_t v = orc_rng_bits(r);
  while (v >= reject_above) v = orc_rng_bits(r);
  return lo + v % span;
}

/* rng.hpp:44-57 (Box-Muller, one engine pair feeds two variates) */
double orc_rng_normal(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  const double u2 = orc_rng_uniform(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double two_pi = 6.283185307179586476925286766559;
  r->spare = radius * sin(two_pi * u2);
  r->have_spare = 1;
  return radius * cos(two_pi * u2);
}

void orc_rng_fill_symmetric(uint64_t seed, int64_t n, double* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_uniform_symmetric(&r);
}

void orc_gaussian_matrix(int64_t m, int64_t n, uint64_t seed, double* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) out[i + j * m] = orc_rng_normal(&r);
}

/* ======================================================================
 * .bed codes -- genio.cpp:33 (code order 00,01,10,11 -> 2, missing, 1, 0)
 * ==================================================================== */
static const uint8_t kCodeToDosage[4] = {2, 3, 1, 0};
static const uint8_t kDosageToCode[4] = {3, 2, 0, 1};

void orc_bed_decode(const uint8_t* payload, int64_t p, int64_t n, uint8_t* out) {
  const int64_t stride = (n + 3) / 4;
  for (int64_t i = 0; i < p; ++i) {
    const uint8_t* rec = payload + i * stride;
    for (int64_t s = 0; s < n; ++s) out[i * n + s] = kCodeToDosage[(rec[s >> 2] >> (2 * (s & 3))) & 3u];
  }
}

void orc_bed_encode(const uint8_t* dosages, int64_t p, int64_t n, uint8_t* payload) {
  const int64_t stride = (n + 3) / 4;
  memset(payload, 0, (size_t)(p * stride)); /* pad bits stay 00 (genio.cpp:100) */
  for (int64_t i = 0; i < p; ++i)
    for (int64_t s = 0; s < n; ++s)
      payload[i * stride + (s >> 2)] |= (uint8_t)(kDosageToCode[dosages[i * n + s] & 3] << (2 * (s & 3)));
}

/* Marker counts: the packed equivalent of the observed-entry loop of
 * impute_mean (genio.cpp:129-139). */
void orc_marker_counts(const uint8_t* payload, int64_t p, int64_t n, int64_t* counts) {
  const int64_t stride = (n + 3) / 4;
  for (int64_t j = 0; j < p; ++j) {
    int64_t c[4] = {0, 0, 0, 0}; /* by code */
    const uint8_t* rec = payload + j * stride;
    for (int64_t s = 0; s < n; ++s) c[(rec[s >> 2] >> (2 * (s & 3))) & 3u]++;
    counts[4 * j + 0] = c[3]; /* dosage 0 */
    counts[4 * j + 1] = c[2]; /* dosage 1 */
    counts[4 * j + 2] = c[0]; /* dosage 2 */
    counts[4 * j + 3] = c[1]; /* missing  */
  }
}

/* impute_mean + standardize (genio.cpp:124-185), restated on counts:
 *   mu   = observed mean (0 when every entry is missing, genio.cpp:139)
 *   var  = population variance over all n entries of the mean-imputed row
 *          (imputed entries add 0; divisor n, genio.cpp:163-165)
 *   zero variance (fewer than two distinct observed dosages) -> zero row,
 *          inv_s = 0 (genio.cpp:167-171)
 *   unit:     s = sqrt(var)                                 (genio.cpp:174-175)
 *   binomial: s = sqrt(q(1-q)), q = clamp(mu/2, 1/(2n+2))   (genio.cpp:176-180)
 *   hwe:      s = sqrt(2 f (1-f)), f = mu/2  (BASELINE.json config standardization)
 *   none:     inv_s = 1, mu = 0: the raw mean-imputed dosages of the
 *             reference CLI's --standardize none (missing -> observed mean,
 *             via orc_geno.mean)
 * The operator entry is (d - mu) * inv_s; the reference divides by s, which
 * differs by at most one rounding per entry. */
void orc_marker_scaling(const int64_t* counts, int64_t p, int64_t n, int scheme, double* mu,
                        double* inv_s) {
  const double nd = (double)n;
  for (int64_t j = 0; j < p; ++j) {
    const int64_t n0 = counts[4 * j], n1 = counts[4 * j + 1], n2 = counts[4 * j + 2];
    const int64_t obs = n0 + n1 + n2;
    if (scheme == ORC_SCALE_NONE) {
      mu[j] = 0.0;
      inv_s[j] = 1.0;
      continue;
    }
    const double m = obs > 0 ? (double)(n1 + 2 * n2) / (double)obs : 0.0;
    mu[j] = m;
    const int distinct = (n0 > 0) + (n1 > 0) + (n2 > 0);
    if (distinct < 2) {
      inv_s[j] = 0.0;
      continue;
    }
    double s;
    if (scheme == ORC_SCALE_UNIT) {
      const double a = 0.0 - m, b = 1.0 - m, c = 2.0 - m;
      const double ss = (double)n0 * (a * a) + (double)n1 * (b * b) + (double)n2 * (c * c);
      s = sqrt(ss / nd);
    } else if (scheme == ORC_SCALE_BINOMIAL) {
      const double clamp = 1.0 / (2.0 * nd + 2.0);
      double q = m / 2.0;
      if (q < clamp) q = clamp;
      if (q > 1.0 - clamp) q = 1.0 - clamp;
      s = sqrt(q * (1.0 - q));
    } else {
      const double f = m / 2.0;
      s = sqrt(2.0 * f * (1.0 - f));
    }
    inv_s[j] = s > 0.0 ? 1.0 / s : 0.0;
  }
}

/* ======================================================================
 * Operators -- linop.hpp:13-117, linop.cpp:9-39
 * ==================================================================== */
static void dense_apply(const orc_op* op, const double* x, double* y) {
  const double* X = (const double*)op->ctx;
  const int64_t m = op->rows, n = op->cols;
  for (int64_t i = 0; i < m; ++i) y[i] = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    const double xj = x[j];
    const double* col = X + j * m;
    for (int64_t i = 0; i < m; ++i) y[i] += col[i] * xj;
  }
}

static void dense_apply_adjoint(const orc_op* op, const double* x, double* y) {
  const double* X = (const double*)op->ctx;
  const int64_t m = op->rows, n = op->cols;
  for (int64_t j = 0; j < n; ++j) {
    const double* col = X + j * m;
    double acc = 0.0;
    for (int64_t i = 0; i < m; ++i) acc += col[i] * x[i];
    y[j] = acc;
  }
}

void orc_dense_op(orc_op* op, const double* X, int64_t m, int64_t n) {
  op->rows = m;
  op->cols = n;
  op->ctx = (void*)X;
  op->apply = dense_apply;
  op->apply_adjoint = dense_apply_adjoint;
}

void orc_marker_means(const int64_t* counts, int64_t p, double* mean) {
  for (int64_t j = 0; j < p; ++j) {
    const int64_t n1 = counts[4 * j + 1], n2 = counts[4 * j + 2];
    const int64_t obs = counts[4 * j] + n1 + n2;
    mean[j] = obs > 0 ? (double)(n1 + 2 * n2) / (double)obs : 0.0;
  }
}

/* One marker's dot product: sum over samples of (d - mu) x_s, a missing
 * entry taking the imputed value `imp` (its mean; genio.cpp:144). */
static double geno_row_dot(const uint8_t* rec, int64_t n, double mu, double imp, const double* x) {
  double acc = 0.0;
  const double vmiss = imp - mu; /* 0 for the standardizing schemes */
  for (int64_t s = 0; s < n; ++s) {
    const unsigned code = (rec[s >> 2] >> (2 * (s & 3))) & 3u;
    if (code == 1u) {
      if (vmiss != 0.0) acc += vmiss * x[s];
      continue;
    }
    acc += ((double)kCodeToDosage[code] - mu) * x[s];
  }
  return acc;
}

void orc_geno_apply_rows(const orc_geno* g, int64_t j0, int64_t j1, const double* x, double* y) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(g->nthreads > 1 ? g->nthreads : 1)
#endif
  for (int64_t j = j0; j < j1; ++j)
    y[j - j0] = geno_row_dot(g->payload + j * g->stride, g->n, g->mu[j],
                             g->mean ? g->mean[j] : g->mu[j], x) * g->inv_s[j];
}

void orc_geno_apply(const orc_geno* g, const double* x, double* y) {
  orc_geno_apply_rows(g, 0, g->p, x, y);
}

/* z_s = sum_j (d_js - mu_j) inv_s_j y_j over observed entries; each thread
 * owns a contiguous sample range and streams every marker in order, so the
 * summation order (marker order) is independent of the thread count. */
void orc_geno_apply_adjoint_rows(const orc_geno* g, int64_t j0, int64_t j1, const double* y,
                                 double* z) {
  const int64_t n = g->n, nbytes = g->stride;
  int nt = g->nthreads > 1 ? g->nthreads : 1;
  for (int64_t s = 0; s < n; ++s) z[s] = 0.0;
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
  {
    int t = 0, T = 1;
#ifdef _OPENMP
    t = omp_get_thread_num();
    T = omp_get_num_threads();
#endif
    const int64_t b0 = nbytes * t / T, b1 = nbytes * (t + 1) / T;
    for (int64_t j = j0; j < j1; ++j) {
      const double w = g->inv_s[j] * y[j - j0];
      const double mu = g->mu[j];
      const double imp = g->mean ? g->mean[j] : mu;
      const double v[4] = {(2.0 - mu) * w, (imp - mu) * w, (1.0 - mu) * w, (0.0 - mu) * w};
      const uint8_t* rec = g->payload + j * g->stride;
      for (int64_t b = b0; b < b1; ++b) {
        const unsigned byte = rec[b];
        const int64_t s0 = 4 * b;
        for (int k = 0; k < 4 && s0 + k < n; ++k) {
          const unsigned code = (byte >> (2 * k)) & 3u;
          if (code != 1u || v[1] != 0.0) z[s0 + k] += v[code];
        }
      }
    }
  }
  (void)nt;
}

void orc_geno_apply_adjoint(const orc_geno* g, const double* y, double* z) {
  orc_geno_apply_adjoint_rows(g, 0, g->p, y, z);
}

static void geno_apply_cb(const orc_op* op, const double* x, double* y) {
  orc_geno_apply((const orc_geno*)op->ctx, x, y);
}
static void geno_apply_adjoint_cb(const orc_op* op, const double* x, double* y) {
  orc_geno_apply_adjoint((const orc_geno*)op->ctx, x, y);
}

void orc_geno_op(orc_op* op, orc_geno* g) {
  g->stride = (g->n + 3) / 4;
  op->rows = g->p;
  op->cols = g->n;
  op->ctx = g;
  op->apply = geno_apply_cb;
  op->apply_adjoint = geno_apply_adjoint_cb;
}

static double vnorm(const double* v, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

static double vdot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* linop.cpp:9-28 */
double orc_norm_estimate(const orc_op* op, int iters, uint64_t seed) {
  const int64_t n = op->cols, m = op->rows;
  if (n == 0 || m == 0) return 0.0;
  orc_rng rng;
  orc_rng_init(&rng, seed);
  double* z = xcalloc((size_t)n, sizeof(double));
  double* y = xcalloc((size_t)m, sizeof(double));
  double* w = xcalloc((size_t)n, sizeof(double));
  for (int64_t i = 0; i < n; ++i) z[i] = orc_rng_uniform_symmetric(&rng);
  double zn = vnorm(z, n);
  if (zn == 0.0) z[0] = zn = 1.0;
  for (int64_t i = 0; i < n; ++i) z[i] /= zn;
  double result = -1.0;
  for (int it = 0; it < iters; ++it) {
    op->apply(op, z, y);
    op->apply_adjoint(op, y, w);
    const double wn = vnorm(w, n);
    if (wn == 0.0) {
      result = 0.0;
      break;
    }
    for (int64_t i = 0; i < n; ++i) z[i] = w[i] / wn;
  }
  if (result < 0.0) {
    op->apply(op, z, y);
    result = vnorm(y, m);
  }
  free(z);
  free(y);
  free(w);
  return result;
}

/* linop.cpp:30-39 */
double orc_adjoint_mismatch(const orc_op* op, uint64_t seed) {
  orc_rng rng;
  orc_rng_init(&rng, seed);
  const int64_t n = op->cols, m = op->rows;
  double* v = xcalloc((size_t)n, sizeof(double));
  double* u = xcalloc((size_t)m, sizeof(double));
  double* xv = xcalloc((size_t)m, sizeof(double));
  double* xtu = xcalloc((size_t)n, sizeof(double));
  for (int64_t i = 0; i < n; ++i) v[i] = orc_rng_normal(&rng);
  for (int64_t i = 0; i < m; ++i) u[i] = orc_rng_normal(&rng);
  op->apply(op, v, xv);
  op->apply_adjoint(op, u, xtu);
  const double left = vdot(u, xv, m), right = vdot(xtu, v, n);
  const double scale = vnorm(u, m) * vnorm(v, n);
  free(v);
  free(u);
  free(xv);
  free(xtu);
  return scale == 0.0 ? 0.0 : fabs(left - right) / scale;
}

/* ======================================================================
 * cgs2 -- orth.hpp:11-44 (eta = 1/sqrt(2))
 * ==================================================================== */
static const double kCgs2Eta = 0.70710678118654752440;

double orc_cgs2(const double* basis, int64_t len, int64_t ncols, double* v, double* coeffs) {
  const double norm_before = vnorm(v, len);
  if (ncols == 0) return norm_before;
  double* c = xcalloc((size_t)ncols, sizeof(double));
  for (int64_t i = 0; i < ncols; ++i) c[i] = vdot(basis + i * len, v, len);
  for (int64_t i = 0; i < ncols; ++i) {
    const double ci = c[i];
    const double* q = basis + i * len;
    for (int64_t r = 0; r < len; ++r) v[r] -= q[r] * ci;
  }
  double norm_after = vnorm(v, len);
  if (norm_after < kCgs2Eta * norm_before) {
    double* c2 = xcalloc((size_t)ncols, sizeof(double));
    for (int64_t i = 0; i < ncols; ++i) c2[i] = vdot(basis + i * len, v, len);
    for (int64_t i = 0; i < ncols; ++i) {
      const double ci = c2[i];
      const double* q = basis + i * len;
      for (int64_t r = 0; r < len; ++r) v[r] -= q[r] * ci;
    }
    for (int64_t i = 0; i < ncols; ++i) c[i] += c2[i];
    free(c2);
    norm_after = vnorm(v, len);
  }
  if (coeffs)
    for (int64_t i = 0; i < ncols; ++i) coeffs[i] += c[i];
  free(c);
  return norm_after;
}

/* ======================================================================
 * svd_small -- small_svd.cpp:14-28. SPEC.md's design decision names
 * one-sided Jacobi; this is Hestenes' method with the de Rijk cyclic order.
 * ==================================================================== */
/* Tall case: A is r x c, r >= c. */
static void jacobi_tall(const double* M, int64_t r, int64_t c, double* U, double* s, double* V) {
  double* A = xcalloc((size_t)(r * c), sizeof(double));
  double* W = xcalloc((size_t)(c * c), sizeof(double));
  memcpy(A, M, sizeof(double) * (size_t)(r * c));
  for (int64_t i = 0; i < c; ++i) W[i + i * c] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    int rotated = 0;
    for (int64_t p = 0; p + 1 < c; ++p) {
      for (int64_t q = p + 1; q < c; ++q) {
        double* ap = A + p * r;
        double* aq = A + q * r;
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int64_t i = 0; i < r; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || fabs(gamma) <= ORC_EPS * sqrt(alpha) * sqrt(beta)) continue;
        rotated = 1;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int64_t i = 0; i < r; ++i) {
          const double x = ap[i], y = aq[i];
          ap[i] = cs * x - sn * y;
          aq[i] = sn * x + cs * y;
        }
        double* wp = W + p * c;
        double* wq = W + q * c;
        for (int64_t i = 0; i < c; ++i) {
          const double x = wp[i], y = wq[i];
          wp[i] = cs * x - sn * y;
          wq[i] = sn * x + cs * y;
        }
      }
    }
    if (!rotated) break;
  }
  /* singular values and descending order (stable) */
  double* sv = xcalloc((size_t)c, sizeof(double));
  int64_t* order = xcalloc((size_t)c, sizeof(int64_t));
  for (int64_t i = 0; i < c; ++i) {
    sv[i] = vnorm(A + i * r, r);
    order[i] = i;
  }
  for (int64_t i = 1; i < c; ++i) {
    const int64_t key = order[i];
    int64_t k = i - 1;
    while (k >= 0 && sv[order[k]] < sv[key]) {
      order[k + 1] = order[k];
      --k;
    }
    order[k + 1] = key;
  }
  const double smax = c > 0 ? sv[order[0]] : 0.0;
  const double zero_tol = smax * ORC_EPS * (double)(r > c ? r : c);
  for (int64_t i = 0; i < c; ++i) {
    const int64_t src = order[i];
    s[i] = sv[src];
    memcpy(V + i * c, W + src * c, sizeof(double) * (size_t)c);
    double* u = U + i * r;
    if (sv[src] > zero_tol && sv[src] > 0.0) {
      for (int64_t k = 0; k < r; ++k) u[k] = A[src * r + k] / sv[src];
    } else {
      /* numerically null direction: orthonormal completion against the
       * columns already placed (classical Gram-Schmidt, twice). */
      int placed = 0;
      for (int64_t e = 0; e < r && !placed; ++e) {
        for (int64_t k = 0; k < r; ++k) u[k] = (k == e) ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
          for (int64_t l = 0; l < i; ++l) {
            const double d = vdot(U + l * r, u, r);
            for (int64_t k = 0; k < r; ++k) u[k] -= d * U[l * r + k];
          }
        const double nn = vnorm(u, r);
        if (nn > 0.5) {
          for (int64_t k = 0; k < r; ++k) u[k] /= nn;
          placed = 1;
        }
      }
    }
  }
  free(sv);
  free(order);
  free(A);
  free(W);
}

int orc_svd_small(const double* M, int64_t r, int64_t c, double* U, double* s, double* V) {
  if (r <= 0 || c <= 0) return 0;
  if (r >= c) {
    jacobi_tall(M, r, c, U, s, V);
    return 0;
  }
  /* wide: M^T = U' S V'^T  =>  M = V' S U'^T */
  double* T = xcalloc((size_t)(r * c), sizeof(double));
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < c; ++j) T[j + i * c] = M[i + j * r];
  jacobi_tall(T, c, r, V, s, U);
  free(T);
  return 0;
}

/* ======================================================================
 * GKL -- gkl.cpp
 * ==================================================================== */
/* gkl.cpp:16-25 */
static double breakdown_factor(void) { return pow(ORC_EPS, 2.0 / 3.0); }
static double one_sided_guard(void) { return 1.0 / sqrt(ORC_EPS); }
static double eps_level(int64_t m, int64_t n) { return ORC_EPS * sqrt((double)(m > n ? m : n)); }

static int monitors_side(int left, int64_t m, int64_t n, const orc_gkl_options* o, double norm_scale) {
  if (!o->one_sided || norm_scale > one_sided_guard()) return 1;
  return left ? (m <= n) : (n < m);
}

void orc_gkl_options_default(orc_gkl_options* o) {
  o->k = 10;
  o->tol = 1e-8;
  o->max_mvps = 1000000;
  o->reorth = ORC_REORTH_PARTIAL;
  o->omega = 1e-8;
  o->one_sided = 0;
  o->restart = ORC_RESTART_NONE;
  o->max_subspace = 40;
  o->keep = 20;
  o->seed = 0;
  o->record_history = 0;
  o->omega_recurrence = 1;
}

/* gkl.cpp:53-73 */
int orc_gkl_options_validate(const orc_gkl_options* o, int64_t m, int64_t n, char* msg, size_t msglen) {
  const int64_t minmn = m < n ? m : n;
  const char* err = NULL;
  if (m <= 0 || n <= 0)
    err = "svdl: operator has an empty dimension";
  else if (o->k < 1 || o->k > minmn)
    err = "svdl: k must lie in [1, min(m, n)]";
  else if (!(o->tol > 0.0))
    err = "svdl: tol must be positive";
  else if (o->max_mvps < 2)
    err = "svdl: max_mvps must allow at least one step";
  else if (o->reorth == ORC_REORTH_PARTIAL && !(o->omega > 0.0))
    err = "svdl: omega must be positive";
  else if (o->restart == ORC_RESTART_THICK) {
    if (o->keep < o->k)
      err = "svdl: keep must be at least k";
    else if (o->keep >= o->max_subspace)
      err = "svdl: keep must be below max_subspace";
    else if (o->max_subspace > minmn)
      err = "svdl: max_subspace cannot exceed min(m, n)";
  }
  if (err) {
    if (msg && msglen) snprintf(msg, msglen, "%s", err);
    return 1;
  }
  return 0;
}

/* gkl.cpp:75-98 */
int orc_lanczos_init(orc_lanczos* f, int64_t m, int64_t n, int64_t capacity, const double* start) {
  memset(f, 0, sizeof(*f));
  if (m <= 0 || n <= 0) return 1;
  int64_t minmn = m < n ? m : n;
  f->m = m;
  f->n = n;
  f->cap = capacity < minmn ? capacity : minmn;
  if (f->cap < 1) return 2;
  const double nrm = vnorm(start, n);
  if (!(nrm > 0.0)) return 3;
  const int64_t cap = f->cap;
  f->U = xcalloc((size_t)(m * cap), sizeof(double));
  f->V = xcalloc((size_t)(n * (cap + 1)), sizeof(double));
  f->B = xcalloc((size_t)(cap * cap), sizeof(double));
  f->coupling = xcalloc((size_t)cap, sizeof(double));
  f->mu = xcalloc((size_t)(cap + 2), sizeof(double));
  f->mu_next = xcalloc((size_t)(cap + 2), sizeof(double));
  f->nu = xcalloc((size_t)(cap + 1), sizeof(double));
  f->nu_next = xcalloc((size_t)(cap + 1), sizeof(double));
  for (int64_t i = 0; i < n; ++i) f->V[i] = start[i] / nrm;
  f->mu[0] = 1.0;
  f->j = 0;
  f->right_exhausted = 0;
  return 0;
}

void orc_lanczos_free(orc_lanczos* f) {
  free(f->U);
  free(f->V);
  free(f->B);
  free(f->coupling);
  free(f->mu);
  free(f->mu_next);
  free(f->nu);
  free(f->nu_next);
  memset(f, 0, sizeof(*f));
}

#define BIDX(f, i, c) ((i) + (c) * (f)->cap)

/* gkl.cpp:112-176 */
static int partial_reorth_update(orc_lanczos* f, int left, double* cand, double cand_coeff,
                                 const orc_gkl_options* o, double norm_scale) {
  const int64_t j = f->j;
  const double lvl = eps_level(f->m, f->n);
  const double tau = 2.0 * lvl * norm_scale + lvl;
  const double denom = cand_coeff > tau + ORC_EPS ? cand_coeff : tau + ORC_EPS;
  double worst = 0.0;
  if (left) {
    for (int64_t i = 0; i < j; ++i) {
      double acc = 0.0;
      for (int64_t c = i; c < j; ++c) acc += fabs(f->B[BIDX(f, i, c)]) * f->mu[c];
      if (o->omega_recurrence == 1) {
        /* alpha u_new = X v - sum_c coupling_c u_c: the u_i component of
         * coupling_c u_c (c != i) is bounded by coupling_c * nu, with nu the
         * committed level of the newest u (or the post-restart carry). */
        for (int64_t c = 0; c < j; ++c)
          if (c != i && f->coupling[c] != 0.0)
            acc += fabs(f->coupling[c]) * f->nu[c > i ? i : c];
      }
      double est = (acc + tau) / denom;
      if (est > 1.0) est = 1.0;
      f->nu_next[i] = est;
      if (est > worst) worst = est;
    }
    f->nu_next[j] = 1.0;
    if (worst > o->omega && monitors_side(1, f->m, f->n, o, norm_scale)) {
      orc_cgs2(f->U, f->m, j, cand, NULL);
      for (int64_t i = 0; i < j; ++i) f->nu_next[i] = lvl;
      return 1;
    }
    return 0;
  }
  const double alpha_last = f->B[BIDX(f, j - 1, j - 1)];
  for (int64_t i = 0; i < j; ++i) {
    double acc = 0.0;
    if (i == j - 1) {
      for (int64_t r = 0; r + 1 < j; ++r) acc += fabs(f->B[BIDX(f, r, i)]) * f->nu[r];
    } else {
      for (int64_t r = 0; r <= i; ++r) acc += fabs(f->B[BIDX(f, r, i)]) * f->nu[r];
      acc += alpha_last * f->mu[i];
    }
    double est = (acc + tau) / denom;
    if (est > 1.0) est = 1.0;
    f->mu_next[i] = est;
    if (est > worst) worst = est;
  }
  f->mu_next[j] = 1.0;
  if (worst > o->omega && monitors_side(0, f->m, f->n, o, norm_scale)) {
    orc_cgs2(f->V, f->n, j, cand, NULL);
    for (int64_t i = 0; i < j; ++i) f->mu_next[i] = lvl;
    return 1;
  }
  return 0;
}

/* gkl.cpp:178-204 */
void orc_deflate_right(orc_lanczos* f, orc_rng* rng) {
  const int64_t j = f->j, n = f->n;
  const double lvl = eps_level(f->m, f->n);
  for (int64_t i = 0; i < j; ++i) f->coupling[i] = 0.0;
  double* V = f->V;
  if (j < n) {
    double* v = xcalloc((size_t)n, sizeof(double));
    for (int attempt = 0; attempt < 4; ++attempt) {
      for (int64_t i = 0; i < n; ++i) v[i] = orc_rng_uniform_symmetric(rng);
      const double nrm = orc_cgs2(V, n, j, v, NULL);
      if (nrm > 1e-3 * sqrt((double)n)) {
        for (int64_t i = 0; i < n; ++i) V[j * n + i] = v[i] / nrm;
        for (int64_t i = 0; i < j; ++i) f->mu[i] = lvl;
        f->mu[j] = 1.0;
        f->right_exhausted = 0;
        free(v);
        return;
      }
    }
    free(v);
  }
  for (int64_t i = 0; i < n; ++i) V[j * n + i] = 0.0;
  for (int64_t i = 0; i <= j; ++i) f->mu[i] = lvl;
  f->right_exhausted = 1;
}

/* gkl.cpp:206-312 */
int orc_bidiag_step(const orc_op* op, orc_lanczos* f, const orc_gkl_options* o, orc_rng* rng,
                    double norm_scale, long* mvp_counter, orc_step_info* info) {
  const int64_t m = f->m, n = f->n, s = f->j;
  const int64_t minmn = m < n ? m : n;
  if (s >= f->cap || s >= minmn) return 1;
  if (f->right_exhausted) return 2;
  memset(info, 0, sizeof(*info));
  info->status = ORC_STEP_OK;
  const double breakdown_tol = breakdown_factor() * norm_scale;
  const double lvl = eps_level(m, n);
  const int full = o->reorth == ORC_REORTH_FULL;
  double* U = f->U;
  double* V = f->V;

  /* Left half-step: alpha u_{s+1} = X v_pending - U coupling. */
  double* w = xcalloc((size_t)m, sizeof(double));
  if (mvp_counter) ++*mvp_counter;
  op->apply(op, V + s * n, w);
  double alpha;
  if (full) {
    alpha = orc_cgs2(U, m, s, w, NULL);
  } else {
    const double w_norm0 = vnorm(w, m);
    for (int64_t i = 0; i < s; ++i)
      if (f->coupling[i] != 0.0) {
        const double ci = f->coupling[i];
        for (int64_t r = 0; r < m; ++r) w[r] -= ci * U[i * m + r];
      }
    double alpha_cand = vnorm(w, m);
    if (alpha_cand < kCgs2Eta * w_norm0) {
      for (int64_t i = 0; i < s; ++i)
        if (f->coupling[i] != 0.0) {
          const double d = vdot(U + i * m, w, m);
          for (int64_t r = 0; r < m; ++r) w[r] -= d * U[i * m + r];
        }
      alpha_cand = vnorm(w, m);
    }
    if (partial_reorth_update(f, 1, w, alpha_cand, o, norm_scale)) {
      info->reorthogonalized_left = 1;
      alpha_cand = vnorm(w, m);
    }
    alpha = alpha_cand;
  }
  if (!(alpha > breakdown_tol)) {
    info->status = ORC_STEP_BREAKDOWN_ALPHA;
    free(w);
    return 0;
  }
  info->alpha = alpha;
  for (int64_t r = 0; r < m; ++r) w[r] /= alpha;
  memcpy(U + s * m, w, sizeof(double) * (size_t)m);
  for (int64_t i = 0; i < s; ++i) f->B[BIDX(f, i, s)] = f->coupling[i];
  f->B[BIDX(f, s, s)] = alpha;
  if (full) {
    for (int64_t i = 0; i < s; ++i) f->nu[i] = lvl;
    f->nu[s] = 1.0;
  } else {
    for (int64_t i = 0; i <= s; ++i) f->nu[i] = f->nu_next[i];
  }
  f->j = s + 1;

  /* Right half-step: beta v_new = X^T u_{s+1} - alpha v_pending. */
  double* z = xcalloc((size_t)n, sizeof(double));
  if (mvp_counter) ++*mvp_counter;
  op->apply_adjoint(op, w, z);
  double beta;
  if (full) {
    beta = orc_cgs2(V, n, s + 1, z, NULL);
  } else {
    const double z_norm0 = vnorm(z, n);
    for (int64_t r = 0; r < n; ++r) z[r] -= alpha * V[s * n + r];
    double beta_cand = vnorm(z, n);
    if (beta_cand < kCgs2Eta * z_norm0) {
      const double d = vdot(V + s * n, z, n);
      for (int64_t r = 0; r < n; ++r) z[r] -= d * V[s * n + r];
      beta_cand = vnorm(z, n);
    }
    if (partial_reorth_update(f, 0, z, beta_cand, o, norm_scale)) {
      info->reorthogonalized_right = 1;
      beta_cand = vnorm(z, n);
    }
    beta = beta_cand;
  }
  for (int64_t i = 0; i <= s; ++i) f->coupling[i] = 0.0;
  if (!(beta > breakdown_tol)) {
    info->status = ORC_STEP_BREAKDOWN_BETA;
    orc_deflate_right(f, rng);
    free(w);
    free(z);
    return 0;
  }
  info->beta = beta;
  for (int64_t r = 0; r < n; ++r) V[(s + 1) * n + r] = z[r] / beta;
  f->coupling[s] = beta;
  if (full) {
    for (int64_t i = 0; i <= s; ++i) f->mu[i] = lvl;
    f->mu[s + 1] = 1.0;
  } else {
    for (int64_t i = 0; i <= s + 1; ++i) f->mu[i] = f->mu_next[i];
  }
  free(w);
  free(z);
  return 0;
}

void orc_ritz_free(orc_ritz* r) {
  free(r->values);
  free(r->WL);
  free(r->WR);
  free(r->err);
  free(r->err_crude);
  free(r->converged);
  memset(r, 0, sizeof(*r));
}

/* gkl.cpp:314-339 */
int orc_ritz_extract(const orc_lanczos* f, double tol, orc_ritz* out) {
  memset(out, 0, sizeof(*out));
  const int64_t j = f->j;
  out->j = j;
  if (j == 0) return 0;
  double* Bj = xcalloc((size_t)(j * j), sizeof(double));
  for (int64_t c = 0; c < j; ++c)
    for (int64_t r = 0; r < j; ++r) Bj[r + c * j] = f->B[BIDX(f, r, c)];
  out->values = xcalloc((size_t)j, sizeof(double));
  out->WL = xcalloc((size_t)(j * j), sizeof(double));
  out->WR = xcalloc((size_t)(j * j), sizeof(double));
  out->err = xcalloc((size_t)j, sizeof(double));
  out->err_crude = xcalloc((size_t)j, sizeof(double));
  out->converged = xcalloc((size_t)j, sizeof(int));
  orc_svd_small(Bj, j, j, out->WL, out->values, out->WR);
  free(Bj);
  for (int64_t i = 0; i < j; ++i) {
    double acc = 0.0;
    for (int64_t r = 0; r < j; ++r) acc += out->WL[r + i * j] * f->coupling[r];
    out->err_crude[i] = fabs(acc);
    out->err[i] = out->err_crude[i];
  }
  for (int64_t i = 0; i < j; ++i) {
    double gap = INFINITY;
    for (int64_t l = 0; l < j; ++l)
      if (l != i) {
        const double d = fabs(out->values[l] - out->values[i]);
        if (d < gap) gap = d;
      }
    if (j > 1 && gap > 10.0 * out->err_crude[i] && gap > 0.0) {
      const double refined = out->err_crude[i] * out->err_crude[i] / gap;
      out->err[i] = out->err_crude[i] < refined ? out->err_crude[i] : refined;
    }
  }
  const double theta_max = out->values[0];
  for (int64_t i = 0; i < j; ++i) out->converged[i] = out->err[i] <= tol * theta_max;
  return 0;
}

/* dst[:, 0:kc] = src[:, 0:j] * W[:, 0:kc] (len rows, W is j x ldw col-major) */
static void basis_rotate(const double* src, int64_t len, int64_t j, const double* W, int64_t ldw,
                         int64_t kc, double* dst) {
  for (int64_t c = 0; c < kc; ++c) {
    double* d = dst + c * len;
    for (int64_t r = 0; r < len; ++r) d[r] = 0.0;
    for (int64_t l = 0; l < j; ++l) {
      const double wl = W[l + c * ldw];
      const double* sc = src + l * len;
      for (int64_t r = 0; r < len; ++r) d[r] += sc[r] * wl;
    }
  }
}

/* gkl.cpp:341-378 */
int orc_thick_restart(orc_lanczos* f, int64_t keep) {
  const int64_t j = f->j, m = f->m, n = f->n;
  if (keep < 1 || keep >= j) return 1;
  orc_ritz ritz;
  orc_ritz_extract(f, 0.0, &ritz);
  double* rho = xcalloc((size_t)keep, sizeof(double));
  for (int64_t i = 0; i < keep; ++i) {
    double acc = 0.0;
    for (int64_t r = 0; r < j; ++r) acc += ritz.WL[r + i * j] * f->coupling[r];
    rho[i] = acc;
  }
  double* un = xcalloc((size_t)(m * keep), sizeof(double));
  basis_rotate(f->U, m, j, ritz.WL, j, keep, un);
  memcpy(f->U, un, sizeof(double) * (size_t)(m * keep));
  free(un);
  double* vn = xcalloc((size_t)(n * keep), sizeof(double));
  basis_rotate(f->V, n, j, ritz.WR, j, keep, vn);
  memcpy(f->V, vn, sizeof(double) * (size_t)(n * keep));
  free(vn);
  memcpy(f->V + keep * n, f->V + j * n, sizeof(double) * (size_t)n);
  memset(f->B, 0, sizeof(double) * (size_t)(f->cap * f->cap));
  for (int64_t i = 0; i < keep; ++i) f->B[BIDX(f, i, i)] = ritz.values[i];
  memset(f->coupling, 0, sizeof(double) * (size_t)f->cap);
  for (int64_t i = 0; i < keep; ++i) f->coupling[i] = rho[i];
  f->j = keep;
  const double lvl = eps_level(m, n);
  const double scale = sqrt((double)j);
  double mmax = f->mu[0], nmax = f->nu[0];
  for (int64_t i = 1; i < j; ++i) {
    if (f->mu[i] > mmax) mmax = f->mu[i];
    if (f->nu[i] > nmax) nmax = f->nu[i];
  }
  double mu_carry = scale * mmax + lvl, nu_carry = scale * nmax + lvl;
  if (mu_carry > 1.0) mu_carry = 1.0;
  if (nu_carry > 1.0) nu_carry = 1.0;
  for (int64_t i = 0; i < keep; ++i) f->mu[i] = mu_carry;
  f->mu[keep] = 1.0;
  for (int64_t i = 0; i < keep; ++i) f->nu[i] = nu_carry;
  free(rho);
  orc_ritz_free(&ritz);
  return 0;
}

/* gkl.cpp:380-409 */
void orc_compress_exhausted(orc_lanczos* f) {
  const int64_t j = f->j, m = f->m, n = f->n;
  if (j == 0) return;
  double* aug = xcalloc((size_t)(j * (j + 1)), sizeof(double));
  for (int64_t c = 0; c < j; ++c)
    for (int64_t r = 0; r < j; ++r) aug[r + c * j] = f->B[BIDX(f, r, c)];
  for (int64_t r = 0; r < j; ++r) aug[r + j * j] = f->coupling[r];
  double* SU = xcalloc((size_t)(j * j), sizeof(double));
  double* Ss = xcalloc((size_t)j, sizeof(double));
  double* SV = xcalloc((size_t)((j + 1) * j), sizeof(double));
  orc_svd_small(aug, j, j + 1, SU, Ss, SV);
  double* un = xcalloc((size_t)(m * j), sizeof(double));
  basis_rotate(f->U, m, j, SU, j, j, un);
  memcpy(f->U, un, sizeof(double) * (size_t)(m * j));
  free(un);
  double* vn = xcalloc((size_t)(n * j), sizeof(double));
  basis_rotate(f->V, n, j + 1, SV, j + 1, j, vn);
  memcpy(f->V, vn, sizeof(double) * (size_t)(n * j));
  free(vn);
  for (int64_t r = 0; r < n; ++r) f->V[j * n + r] = 0.0;
  memset(f->B, 0, sizeof(double) * (size_t)(f->cap * f->cap));
  for (int64_t i = 0; i < j; ++i) f->B[BIDX(f, i, i)] = Ss[i];
  memset(f->coupling, 0, sizeof(double) * (size_t)f->cap);
  f->right_exhausted = 1;
  const double lvl = eps_level(m, n);
  for (int64_t i = 0; i <= j; ++i) f->mu[i] = lvl;
  for (int64_t i = 0; i < j; ++i) f->nu[i] = lvl;
  free(aug);
  free(SU);
  free(Ss);
  free(SV);
}

/* gkl.cpp:411-414 */
double orc_error_metric_l1(const orc_ritz* r, int64_t k) {
  const int64_t count = k < r->j ? k : r->j;
  double s = 0.0;
  for (int64_t i = 0; i < count; ++i) s += r->err_crude[i];
  return s;
}

void orc_svdl_result_free(orc_svdl_result* r) {
  free(r->singvals);
  free(r->U);
  free(r->V);
  free(r->err);
  free(r->converged);
  free(r->ritz_history);
  free(r->err_history);
  memset(r, 0, sizeof(*r));
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct {
  const orc_gkl_options* o;
  orc_svdl_result* res;
  int64_t hist_cap;
} hist_state;

static void record(hist_state* h, const orc_ritz* ritz) {
  orc_svdl_result* res = h->res;
  const int64_t k = h->o->k;
  if (res->history_len == h->hist_cap) {
    h->hist_cap = h->hist_cap ? 2 * h->hist_cap : 64;
    res->ritz_history = realloc(res->ritz_history, sizeof(double) * (size_t)(h->hist_cap * k));
    res->err_history = realloc(res->err_history, sizeof(double) * (size_t)(h->hist_cap * k));
  }
  double* rv = res->ritz_history + res->history_len * k;
  double* ev = res->err_history + res->history_len * k;
  for (int64_t i = 0; i < k; ++i) {
    rv[i] = i < ritz->j ? ritz->values[i] : NAN;
    ev[i] = i < ritz->j ? ritz->err[i] : NAN;
  }
  res->history_len++;
}

/* gkl.cpp:416-514 */
int orc_svdl(const orc_op* op, const orc_gkl_options* o, orc_svdl_result* res, char* msg,
             size_t msglen) {
  const double t_start = now_seconds();
  memset(res, 0, sizeof(*res));
  const int64_t m = op->rows, n = op->cols;
  if (orc_gkl_options_validate(o, m, n, msg, msglen)) return 1;
  const int64_t minmn = m < n ? m : n;
  const int64_t cap = o->restart == ORC_RESTART_THICK ? o->max_subspace : minmn;

  long mvps = 0;
  orc_rng rng;
  orc_rng_init(&rng, o->seed);
  double* v0 = xcalloc((size_t)n, sizeof(double));
  for (int64_t i = 0; i < n; ++i) v0[i] = orc_rng_uniform_symmetric(&rng);
  orc_lanczos f;
  if (orc_lanczos_init(&f, m, n, cap, v0)) {
    free(v0);
    if (msg && msglen) snprintf(msg, msglen, "LanczosFactorization: zero start vector");
    return 2;
  }
  free(v0);

  double norm_scale = 0.0;
  orc_ritz ritz;
  memset(&ritz, 0, sizeof(ritz));
  int consecutive_breakdowns = 0;
  hist_state hs = {o, res, 0};

#define EXTRACT()                                                   \
  do {                                                              \
    orc_ritz_free(&ritz);                                           \
    orc_ritz_extract(&f, o->tol, &ritz);                            \
    if (ritz.j > 0 && ritz.values[0] > norm_scale) norm_scale = ritz.values[0]; \
    if (o->record_history) record(&hs, &ritz);                      \
  } while (0)

#define TOPK_CONVERGED() (topk_converged(&f, &ritz, o->k))

  while (1) {
    if (f.j >= minmn) break;
    if (mvps + 2 > o->max_mvps) break;
    if (f.right_exhausted) break;
    orc_step_info step;
    orc_bidiag_step(op, &f, o, &rng, norm_scale, &mvps, &step);
    if (step.status == ORC_STEP_BREAKDOWN_ALPHA) {
      res->deflations++;
      consecutive_breakdowns++;
      orc_compress_exhausted(&f);
      EXTRACT();
      int conv = 1;
      if (f.j < o->k || ritz.j < o->k) conv = 0;
      else
        for (int64_t i = 0; i < o->k; ++i)
          if (!ritz.converged[i]) conv = 0;
      if (conv || consecutive_breakdowns > 3) break;
      orc_deflate_right(&f, &rng);
      continue;
    }
    res->steps++;
    if (step.reorthogonalized_left) res->reorth_count++;
    if (step.reorthogonalized_right) res->reorth_count++;
    {
      const double h = hypot(step.alpha, step.beta);
      if (h > norm_scale) norm_scale = h;
    }
    if (step.status == ORC_STEP_BREAKDOWN_BETA) {
      res->deflations++;
      consecutive_breakdowns++;
    } else {
      consecutive_breakdowns = 0;
    }
    if (o->restart == ORC_RESTART_NONE) {
      EXTRACT();
      int conv = 1;
      if (f.j < o->k || ritz.j < o->k) conv = 0;
      else
        for (int64_t i = 0; i < o->k; ++i)
          if (!ritz.converged[i]) conv = 0;
      if (conv) break;
    } else if (f.j == o->max_subspace) {
      EXTRACT();
      int conv = 1;
      if (f.j < o->k || ritz.j < o->k) conv = 0;
      else
        for (int64_t i = 0; i < o->k; ++i)
          if (!ritz.converged[i]) conv = 0;
      if (conv) break;
      if (mvps + 2 > o->max_mvps) break;
      orc_thick_restart(&f, o->keep);
      res->restarts++;
    }
  }

  EXTRACT();
  const int64_t j = f.j;
  const int64_t count = o->k < j ? o->k : j;
  res->count = count;
  res->singvals = xcalloc((size_t)count, sizeof(double));
  res->err = xcalloc((size_t)count, sizeof(double));
  res->converged = xcalloc((size_t)count, sizeof(int));
  res->U = xcalloc((size_t)(m * count), sizeof(double));
  res->V = xcalloc((size_t)(n * count), sizeof(double));
  for (int64_t i = 0; i < count; ++i) {
    res->singvals[i] = ritz.values[i];
    res->err[i] = ritz.err[i];
    res->converged[i] = ritz.converged[i];
  }
  if (count > 0) {
    basis_rotate(f.U, m, j, ritz.WL, j, count, res->U);
    basis_rotate(f.V, n, j, ritz.WR, j, count, res->V);
  }
  {
    int conv = 1;
    if (f.j < o->k || ritz.j < o->k) conv = 0;
    else
      for (int64_t i = 0; i < o->k; ++i)
        if (!ritz.converged[i]) conv = 0;
    res->all_converged = (count == o->k) && conv;
  }
  res->mvps = mvps;
  res->wall_seconds = now_seconds() - t_start;
  orc_ritz_free(&ritz);
  orc_lanczos_free(&f);
#undef EXTRACT
#undef TOPK_CONVERGED
  return 0;
}

/* ======================================================================
 * Synthetic genotypes: counter-based draws keyed by (seed, marker, sample)
 * so that any shard or sub-block regenerates identically on CPU and GPU.
 * Definition shared with paper_1808_03374_b200/csrc/synth.cu.
 * ==================================================================== */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline double u53(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

static inline uint64_t marker_key(uint64_t seed, int64_t j) {
  return mix64(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)j + 1ULL);
}
static inline uint64_t cell_key(uint64_t mk, int64_t i) {
  return mix64(mk ^ ((uint64_t)i * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
}

static double sample_freq(const orc_synth_spec* s, int64_t j, int64_t i) {
  if (s->pop) return s->freq[(int64_t)s->pop[i] * s->p + j];
  double acc = 0.0;
  for (int k = 0; k < s->npop; ++k) acc = acc + s->admix[i * s->npop + k] * s->freq[(int64_t)k * s->p + j];
  return acc;
}

static int draw_dosage(const orc_synth_spec* s, uint64_t mk, int64_t j, int64_t i) {
  const uint64_t h = cell_key(mk, i);
  const double f = sample_freq(s, j, i);
  int d = (u53(mix64(h + 1)) < f) + (u53(mix64(h + 2)) < f);
  if (s->copy_from && s->copy_from[i] >= 0 && u53(mix64(h + 4)) < s->copy_prob) {
    const int64_t a = s->copy_from[i];
    const uint64_t ha = cell_key(mk, a);
    const double fa = sample_freq(s, j, a);
    d = (u53(mix64(ha + 1)) < fa) + (u53(mix64(ha + 2)) < fa);
  }
  if (s->missing_rate > 0.0 && u53(mix64(h + 3)) < s->missing_rate) return 3;
  return d;
}

void orc_synth_bed(const orc_synth_spec* s, int64_t j0, int64_t j1, uint8_t* out) {
  const int64_t n = s->n, stride = (n + 3) / 4;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int64_t j = j0; j < j1; ++j) {
    uint8_t* rec = out + (j - j0) * stride;
    memset(rec, 0, (size_t)stride);
    const uint64_t mk = marker_key(s->seed, j);
    for (int64_t i = 0; i < n; ++i)
      rec[i >> 2] |= (uint8_t)(kDosageToCode[draw_dosage(s, mk, j, i)] << (2 * (i & 3)));
  }
}
