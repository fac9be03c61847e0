/*
 * gkb_oracle.h -- CPU restatement of the reference's GKL hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in paper_1808_03374_b200/ may include,
 * link or call this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg use it, as the checker and the CPU
 * baseline. The product path has no CPU fallback.
 *
 * Restates (file:line under /root/reference):
 *   proj/include/gkpca/rng.hpp:17-62      Rng (mt19937_64 + draw algorithms)
 *   proj/src/genio.cpp:33,53-83           .bed 2-bit decode
 *   proj/src/genio.cpp:124-185            impute_mean + standardize semantics
 *   proj/include/gkpca/linop.hpp:13-117   LinearOperator / counting
 *   proj/src/linop.cpp:9-39               norm_estimate, adjoint_mismatch
 *   proj/include/gkpca/orth.hpp:11-44     cgs2
 *   proj/src/small_svd.cpp:14-28          svd_small (one-sided Jacobi)
 *   proj/src/gkl.cpp:16-514               GKL driver (svdl and helpers)
 *
 * Parity pinning: the reference cannot be compiled here (Eigen3 and vendor/
 * are absent), so this restatement is pinned on
 * the reference's own known-answer tests (proj/tests/test_gkl.cpp,
 * test_linops.cpp, test_genio.cpp) and property tests against LAPACK SVD, see
 * tests/test_oracle_*.py.
 *
 * Conventions: dense matrices are column-major (Eigen default), fp64.
 * Genotype matrices are .bed payloads: p marker records of ceil(n/4) bytes,
 * reference orientation X = p x n (markers are rows).
 */
#ifndef GKB_ORACLE_H
#define GKB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- Rng: rng.hpp:17-62 ------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int mti;
  double spare;
  int have_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_bits(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_uniform_symmetric(orc_rng* r);
uint64_t orc_rng_uniform_int(orc_rng* r, uint64_t lo, uint64_t hi);
double orc_rng_normal(orc_rng* r);
/* Fills out[i] = uniform_symmetric() for i < n (gkl.cpp:427-429). */
void orc_rng_fill_symmetric(uint64_t seed, int64_t n, double* out);
/* Fills a column-major m x n matrix with normal() column by column
 * (tests/oracles.hpp:157-163, gaussian_matrix). */
void orc_gaussian_matrix(int64_t m, int64_t n, uint64_t seed, double* out);

/* ---- .bed decode and marker statistics: genio.cpp:33,124-185 ----------- */
/* Decodes marker-major payload to dosages (3 = missing), out is p x n
 * row-major (marker i, sample s at out[i*n+s]). */
void orc_bed_decode(const uint8_t* payload, int64_t p, int64_t n, uint8_t* out);
/* Packs dosages (row-major p x n, 3 = missing) to a payload, pads 00
 * (genio.cpp:85-122). */
void orc_bed_encode(const uint8_t* dosages, int64_t p, int64_t n, uint8_t* payload);

enum { ORC_SCALE_UNIT = 0, ORC_SCALE_BINOMIAL = 1, ORC_SCALE_HWE = 2, ORC_SCALE_NONE = 3 };
/* Per-marker counts [n0, n1, n2, nmiss] (int64 x 4 per marker). */
void orc_marker_counts(const uint8_t* payload, int64_t p, int64_t n, int64_t* counts);
/* mu (observed mean, 0 for an all-missing marker) and inv_s (1/scale, 0 for
 * zero-variance markers) from counts; scheme per ORC_SCALE_*. */
void orc_marker_scaling(const int64_t* counts, int64_t p, int64_t n, int scheme,
                        double* mu, double* inv_s);

/* ---- operators: linop.hpp:13-117 --------------------------------------- */
typedef struct orc_op {
  int64_t rows, cols;
  void* ctx;
  void (*apply)(const struct orc_op* op, const double* x, double* y);         /* y = X x   */
  void (*apply_adjoint)(const struct orc_op* op, const double* x, double* y); /* y = X^T x */
} orc_op;

/* Dense column-major m x n operator (DenseOperator, linop.hpp:43-64). The
 * matrix is borrowed. */
void orc_dense_op(orc_op* op, const double* X, int64_t m, int64_t n);

/* Packed standardized genotype operator: entry (j,s) = (d_js - mu_j)*inv_s_j
 * when observed, (mean_j - mu_j)*inv_s_j when missing (impute_mean, then the
 * affine standardization: genio.cpp:144,182). mean_j is the observed mean
 * (orc_marker_means); for the standardizing schemes mu_j = mean_j and missing
 * entries are 0; mean == NULL means 0 for missing entries. All buffers
 * borrowed. nthreads<=1: one thread. */
typedef struct {
  const uint8_t* payload;
  int64_t p, n, stride;
  const double* mu;
  const double* inv_s;
  int nthreads;
  const double* mean;
} orc_geno;
/* Observed mean per marker from counts [n0,n1,n2,nmiss] (0 when all missing,
 * genio.cpp:139). */
void orc_marker_means(const int64_t* counts, int64_t p, double* mean);
void orc_geno_op(orc_op* op, orc_geno* g);
void orc_geno_apply(const orc_geno* g, const double* x, double* y);
void orc_geno_apply_adjoint(const orc_geno* g, const double* y, double* z);
/* Apply restricted to markers [j0, j1): y[j-j0]; adjoint partial over the
 * same markers, z over all n samples (the shard-local work of a
 * SNP-sharded rank). */
void orc_geno_apply_rows(const orc_geno* g, int64_t j0, int64_t j1, const double* x, double* y);
void orc_geno_apply_adjoint_rows(const orc_geno* g, int64_t j0, int64_t j1, const double* y,
                                 double* z);

double orc_norm_estimate(const orc_op* op, int iters, uint64_t seed); /* linop.cpp:9-28 */
double orc_adjoint_mismatch(const orc_op* op, uint64_t seed);         /* linop.cpp:30-39 */

/* ---- cgs2: orth.hpp:11-44 ---------------------------------------------- */
/* basis: len x ncols column-major; coeffs (may be NULL) receives basis^T v
 * accumulated. Returns ||v|| after; v is not normalized. */
double orc_cgs2(const double* basis, int64_t len, int64_t ncols, double* v, double* coeffs);

/* ---- svd_small: small_svd.cpp:14-28 (one-sided Jacobi, SPEC design) ----- */
/* M is r x c column-major. Outputs: U r x k, s k, V c x k, k = min(r,c),
 * singular values descending, U/V orthonormal columns. Returns 0 on success. */
int orc_svd_small(const double* M, int64_t r, int64_t c, double* U, double* s, double* V);

/* ---- GKL: gkl.hpp:17-196, gkl.cpp -------------------------------------- */
enum { ORC_REORTH_FULL = 0, ORC_REORTH_PARTIAL = 1 };
enum { ORC_RESTART_NONE = 0, ORC_RESTART_THICK = 1 };
enum { ORC_STEP_OK = 0, ORC_STEP_BREAKDOWN_ALPHA = 1, ORC_STEP_BREAKDOWN_BETA = 2 };

typedef struct {
  int64_t k;          /* 10 */
  double tol;         /* 1e-8 */
  int64_t max_mvps;   /* 1000000 */
  int reorth;         /* partial */
  double omega;       /* 1e-8 */
  int one_sided;      /* 0 */
  int restart;        /* none */
  int64_t max_subspace; /* 40 */
  int64_t keep;       /* 20 */
  uint64_t seed;      /* 0 */
  int record_history; /* 0 */
  /* Left omega recurrence: 0 = as written in gkl.cpp:127-136, which omits the
   * previous-level term |coupling_c| * nu; 1 = complete recurrence (adds it,
   * mirroring the right-side recurrence's alpha_last * mu term, :155-160). */
  int omega_recurrence;
} orc_gkl_options;

void orc_gkl_options_default(orc_gkl_options* o);
/* Returns 0 when valid, else nonzero and fills msg (gkl.cpp:53-73). */
int orc_gkl_options_validate(const orc_gkl_options* o, int64_t m, int64_t n, char* msg, size_t msglen);

typedef struct {
  int64_t m, n, cap, j;
  double* U;        /* m x cap   */
  double* V;        /* n x (cap+1) */
  double* B;        /* cap x cap */
  double* coupling; /* cap */
  double* mu;       /* cap+2 */
  double* nu;       /* cap+1 */
  double* mu_next;  /* cap+2 */
  double* nu_next;  /* cap+1 */
  int right_exhausted;
} orc_lanczos;

/* LanczosFactorization ctor (gkl.cpp:75-98); returns 0 or nonzero on error. */
int orc_lanczos_init(orc_lanczos* f, int64_t m, int64_t n, int64_t capacity, const double* start);
void orc_lanczos_free(orc_lanczos* f);

typedef struct {
  int status;
  int reorthogonalized_left, reorthogonalized_right;
  double alpha, beta;
} orc_step_info;

/* bidiag_step (gkl.cpp:206-312). Returns 0, or nonzero on a logic error
 * (factorization full / right side exhausted). */
int orc_bidiag_step(const orc_op* op, orc_lanczos* f, const orc_gkl_options* o, orc_rng* rng,
                    double norm_scale, long* mvp_counter, orc_step_info* info);

typedef struct {
  int64_t j;
  double* values;   /* j */
  double* WL;       /* j x j */
  double* WR;       /* j x j */
  double* err;      /* j */
  double* err_crude;/* j */
  int* converged;   /* j */
} orc_ritz;
int orc_ritz_extract(const orc_lanczos* f, double tol, orc_ritz* out);
void orc_ritz_free(orc_ritz* r);
int orc_thick_restart(orc_lanczos* f, int64_t keep);
void orc_compress_exhausted(orc_lanczos* f);
void orc_deflate_right(orc_lanczos* f, orc_rng* rng);
double orc_error_metric_l1(const orc_ritz* r, int64_t k);

typedef struct {
  int64_t count;       /* min(k, steps) */
  double* singvals;    /* count */
  double* U;           /* m x count */
  double* V;           /* n x count */
  double* err;         /* count */
  int* converged;      /* count */
  long mvps;
  int64_t steps;
  int restarts, reorth_count, deflations, all_converged;
  double wall_seconds;
  int64_t history_len;   /* extractions recorded */
  double* ritz_history;  /* history_len x k (padded with NaN) */
  double* err_history;
} orc_svdl_result;

/* svdl (gkl.cpp:416-514). Returns 0, or nonzero on invalid options (msg). */
int orc_svdl(const orc_op* op, const orc_gkl_options* o, orc_svdl_result* res, char* msg,
             size_t msglen);
void orc_svdl_result_free(orc_svdl_result* r);

/* ---- synthetic genotypes (counter-based; shared definition with the
 * device generator, see paper_1808_03374_b200/csrc/synth.cu) ------------- */
typedef struct {
  int64_t p, n;
  uint64_t seed;
  int npop;              /* subpopulations */
  const double* freq;    /* npop x p, freq[k*p + j] (drawn host-side) */
  const int32_t* pop;    /* n: subpopulation of each sample, or NULL when admixed */
  const double* admix;   /* n x npop mixing weights (row i), used when pop == NULL */
  double missing_rate;
  const int32_t* copy_from; /* n: sample whose genotypes this one copies
                               (with probability copy_prob per marker), -1 none;
                               NULL when there are no related pairs */
  double copy_prob;
} orc_synth_spec;
/* Writes the .bed payload for markers [j0, j1) into out (rows j0..j1-1). */
void orc_synth_bed(const orc_synth_spec* s, int64_t j0, int64_t j1, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
