/*
 * gkb.h -- C ABI of the B200-native GKL hot path (libgkb.so).
 *
 * The reference (arxiv 1808.03374 C++ library, /root/reference/proj) exposes
 * its hot path through C++ classes; this header is the drop-in boundary a
 * cgo / JNI / ctypes / C++ caller binds instead. Each entry point cites the
 * reference interface it replaces (file:line under /root/reference).
 *
 * Conventions:
 *  - every function returns an int status (GKB_OK = 0); the message of the
 *    last failure on the calling thread is gkb_last_error(). No exception
 *    crosses the ABI; the C++ mirror (paper_1808_03374_b200/gkl.py for Python,
 *    INTEGRATION.md for C++) rethrows with the reference's exception types:
 *    GKB_EINVAL -> std::invalid_argument, GKB_ELOGIC -> std::logic_error,
 *    GKB_EFORMAT -> FormatError.
 *  - orientation follows the reference: an operator is m x n with
 *    apply(x) = X x (x has n entries) and apply_adjoint(y) = X^T y. A genotype
 *    operator is markers x samples (m = p SNPs, n individuals), i.e. the
 *    reference's standardized GenotypeMatrix (genio.hpp:23-32).
 *  - dense matrices are column-major fp64 (Eigen default, types.hpp:13-16).
 *  - handles own all device memory; host buffers are borrowed for the call.
 *  - calls on one context are stream-ordered and not thread-safe (the
 *    reference's single-caller driver).
 */
#ifndef GKB_H
#define GKB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GKB_OK 0
#define GKB_EINVAL 1  /* std::invalid_argument (gkl.cpp:53-73, linop.hpp:103-104) */
#define GKB_ELOGIC 2  /* std::logic_error (gkl.cpp:215-218, :344)                  */
#define GKB_ECUDA 3
#define GKB_ENCCL 4
#define GKB_EOOM 5
#define GKB_EFORMAT 6 /* FormatError (genio.hpp:14-17)                              */

typedef struct gkb_ctx gkb_ctx;
typedef struct gkb_op gkb_op;
typedef struct gkb_lanczos gkb_lanczos;

const char* gkb_last_error(void);
const char* gkb_version(void);

/* ---- context ------------------------------------------------------------
 * A context owns the CUDA streams, the SNP shards and the communicator.
 * gkb_init: one process drives `nshards` shards on devices[i] (devices may
 * repeat, e.g. several shards on one GPU to exercise the sharded path; the
 * cross-shard sums then run as fixed-order device reductions).
 * gkb_init_nccl: one process per GPU (SPMD); rank r owns SNP shard r and the
 * sums run as ncclAllReduce over NVLink. The 128-byte id comes from
 * gkb_nccl_unique_id() on rank 0, broadcast by the caller (torch.distributed). */
int gkb_init(int nshards, const int* devices, gkb_ctx** ctx);
int gkb_nccl_unique_id(uint8_t id_out[128]);
int gkb_init_nccl(int device, const uint8_t id[128], int nranks, int rank, gkb_ctx** ctx);
/* gkb_init_host_comm: SPMD like gkb_init_nccl, with the sums done by the
 * caller: `fn(user, buf, count)` must replace the page-locked host buffer
 * buf[0..count) by its elementwise sum over all ranks (a collective: every
 * rank makes the same calls in the same order). It runs on a CUDA host-
 * function thread between a D2H and an H2D copy on the shard's stream, so it
 * must not call CUDA. Used to run the multi-process path of the library as
 * several processes on ONE GPU (e.g. an allreduce over torch.distributed /
 * gloo), since NCCL cannot place two ranks on one device; no kernel waits
 * on another process. */
typedef void (*gkb_host_allreduce_fn)(void* user, double* buf, int64_t count);
int gkb_init_host_comm(int device, int nranks, int rank, gkb_host_allreduce_fn fn, void* user,
                       gkb_ctx** ctx);
int gkb_destroy(gkb_ctx* ctx);
/* nshards local to this process, world size, this process's first shard index */
int gkb_ctx_info(gkb_ctx* ctx, int* nshards_local, int* nshards_total, int* first_shard);
int gkb_synchronize(gkb_ctx* ctx);

/* Contiguous SNP (operator-row) partition used for sharding: starts[0..nparts]
 * with starts[nparts] = m; interior boundaries are multiples of 4 rows. */
int gkb_partition_rows(int64_t m, int nparts, int64_t* starts);

/* ---- operators (LinearOperator, linop.hpp:13-39) -------------------------- */
/* Packed genotype operator from a .bed payload (the bytes after the 3-byte
 * header; p marker records of ceil(n/4) bytes, code 00->2, 01->missing,
 * 10->1, 11->0; genio.cpp:33,53-83). Uploads and re-lays the 2-bit codes into
 * HBM and counts per-marker dosages on the device. In SPMD mode every rank
 * passes the same full payload pointer (e.g. an mmap) and keeps its rows.
 * Scaling must be set (gkb_geno_standardize / gkb_geno_set_scaling) before
 * applying; the operator entry is (d - mu_j) * inv_s_j, 0 when missing
 * (impute_mean + standardize, genio.cpp:124-185). */
int gkb_geno_from_bed(gkb_ctx* ctx, const uint8_t* payload, int64_t p, int64_t n, gkb_op** op);

/* read_bed's checks (genio.cpp:53-70) without reading the payload: p = non-
 * empty lines of the .bim, n = of the .fam (count_lines, genio.cpp:21-30);
 * magic 6C 1B, mode 01, size == p*ceil(n/4)+3. GKB_EFORMAT with the
 * reference's messages ("cannot open ...", ": bad magic", ": only marker-major
 * mode (0x01) is supported", ": payload size mismatch (expected E bytes,
 * found F)"). Needs no GPU. */
int gkb_bed_check(const char* bed, const char* bim, const char* fam, int64_t* p, int64_t* n);

/* .bed file -> HBM (replaces read_bed + load_matrix, gkpca.cpp:89-108): the
 * checks above, then each shard's records are streamed from the file with
 * positional reads into double-buffered pinned staging, overlapped with the
 * device-side layout builds (each rank / shard reads only its own rows). */
int gkb_geno_from_bed_file(gkb_ctx* ctx, const char* bed, const char* bim, const char* fam,
                           gkb_op** op);

/* Synthetic Balding-Nichols genotypes generated directly on the device with
 * the counter-based draws of oracle/gkb_oracle.c:orc_synth_bed (bit-identical
 * .bed bytes). freq: npop x p (row k at freq[k*p]); pop: n subpopulation ids
 * or NULL with admix (n x npop weights); copy_from: n (-1 = none) or NULL. */
typedef struct {
  int64_t p, n;
  uint64_t seed;
  int npop;
  const double* freq;
  const int32_t* pop;
  const double* admix;
  double missing_rate;
  const int32_t* copy_from;
  double copy_prob;
} gkb_synth_spec;
int gkb_geno_from_synth(gkb_ctx* ctx, const gkb_synth_spec* spec, gkb_op** op);

/* Per-marker [n0, n1, n2, nmissing] (int64, p x 4), counted on the device. */
int gkb_geno_counts(gkb_op* op, int64_t* counts);
/* Per-marker PC-adjusted regression scan (the per-marker fits of gkpca
 * regress, gkpca.cpp:554-680, with regress.cpp:10-65's estimates by
 * Frisch-Waugh-Lovell): for every marker i, y ~ [1, m_i, Z] (Z: n x k,
 * column-major, may be NULL for k = 0). Block product and per-marker algebra
 * on the device; outputs of length p; dep[i] = 1 where the reference reports
 * the rank-deficiency error for design column 1. */
int gkb_geno_marker_scan(gkb_op* op, const double* y, const double* Z, int64_t k, int unbiased,
                         double* beta, double* se, double* intercept, double* sigma2,
                         int32_t* dep);
/* scheme: 0 unit variance (genio.cpp:174-175), 1 binomial with clamp
 * (genio.cpp:176-180), 2 hwe sqrt(2f(1-f)) (BASELINE.json standardization),
 * 3 none (raw dosage, missing -> 0). Computes (mu, inv_s) from the device
 * counts on the host and installs them. */
int gkb_geno_standardize(gkb_op* op, int scheme);
int gkb_geno_set_scaling(gkb_op* op, const double* mu, const double* inv_s);
int gkb_geno_get_scaling(gkb_op* op, double* mu, double* inv_s);
/* Device-memory plan of one shard of p_loc SNPs x n samples at a missing
 * fraction: both tile layouts (one per product) when they fit in free_bytes,
 * else layout 1 only (the adjoint then reads layout 1: single-layout mode,
 * e.g. config 5 at 2 GPUs, 125 GB per layout per GPU). Host-only; the
 * operator builders apply it with the device's free memory (GKB_LAYOUTS=1|2
 * forces a mode). */
int gkb_geno_plan(int64_t p_loc, int64_t n, double missing_fraction, int64_t free_bytes,
                  int* layouts, int64_t* dual_bytes, int64_t* single_bytes);
/* The modes an operator's shards were built in: layouts 1 or 2, and whether
 * the missing entries are handled by indicator MMAs (dense_missing = 1, above
 * 1.5% missing; GKB_MISS_MODE=list|ind forces) instead of per-CTA lists. */
int gkb_geno_layouts(gkb_op* op, int* layouts, int* dense_missing);
/* Reads rows [row0, row0+nrows) back from HBM as .bed records (layout round
 * trip; pads written 00 as write_bed does, genio.cpp:100). */
int gkb_geno_read_bed(gkb_op* op, int64_t row0, int64_t nrows, uint8_t* payload_out);
/* Total missing entries, packed bytes per mvp (sum over shards of
 * p_shard*ceil(n/4)) and device bytes resident. */
int gkb_geno_info(gkb_op* op, int64_t* nmissing, int64_t* packed_bytes, int64_t* device_bytes);

/* DenseOperator (linop.hpp:43-64) on the device: X is m x n column-major. */
int gkb_dense_create(gkb_ctx* ctx, const double* X, int64_t m, int64_t n, gkb_op** op);

int gkb_op_shape(gkb_op* op, int64_t* rows, int64_t* cols);
/* y = X x (apply, linop.hpp:21-22; DenseOperator::apply linop.hpp:50-53) and
 * y = X^T x (apply_adjoint, linop.hpp:25-26 / :55-58) on HOST vectors:
 * H2D, device kernels, cross-shard sum, D2H. Each call counts one mvp
 * (CountingOperator, linop.hpp:72-97). */
int gkb_op_apply(gkb_op* op, const double* x, double* y);
int gkb_op_apply_adjoint(gkb_op* op, const double* x, double* y);
int64_t gkb_op_mvps(gkb_op* op);
/* k columns at once (column-major host blocks, X: cols x k -> Y: rows x k,
 * and Y: rows x k -> Z: cols x k): one H2D, the k products back to back on
 * the device, one D2H; k mvps. The column loops of subspace_iterate
 * (subspace.cpp:70-77, :97-101) call these. */
int gkb_op_apply_block(gkb_op* op, const double* X, int64_t k, double* Y);
int gkb_op_apply_adjoint_block(gkb_op* op, const double* Y, int64_t k, double* Z);
/* Page-locked host memory for the vectors passed to gkb_op_apply /
 * gkb_op_apply_adjoint (no reference counterpart: the reference's vectors are
 * Eigen::VectorXd in pageable memory). Copies from/to these buffers run at
 * full PCIe/C2C DMA rate; any host pointer remains valid input. */
int gkb_host_alloc(size_t bytes, void** ptr);
int gkb_host_free(void* ptr);
int gkb_op_destroy(gkb_op* op);

/* Device-resident timing loop used by bench.py: `iters` applications of
 * which = 0 apply, 1 apply_adjoint, 2 one of each, on device vectors,
 * optionally flushing L2 between iterations. Returns the CUDA-event time per
 * iteration (stream-ordered, whole sequence) and the summed time of the main
 * packed kernels alone (ms). */
int gkb_op_bench(gkb_op* op, int which, int iters, int flush_l2, double* ms_per_iter,
                 double* main_kernel_ms_per_iter, int* launches_per_iter);

/* ---- GKL solver (gkl.hpp:17-196) ----------------------------------------- */
typedef struct {
  int64_t k;            /* 10    */
  double tol;           /* 1e-8  */
  int64_t max_mvps;     /* 1e6   */
  int reorth;           /* 0 full (kFull), 1 partial (kPartial, default) */
  double omega;         /* 1e-8  */
  int one_sided;        /* 0     */
  int restart;          /* 0 none (kNone, default), 1 thick (kThick) */
  int64_t max_subspace; /* 40    */
  int64_t keep;         /* 20    */
  uint64_t seed;        /* 0     */
  int record_history;   /* 0     */
  /* Left-side omega recurrence of partial reorthogonalization:
   * 0 = exactly as written in gkl.cpp:127-136 (omits the |coupling|*nu
   *     previous-level term, so the estimates can under-run the true loss of
   *     orthogonality; the reference's own test_gkl.cpp:124-171 fails);
   * 1 = complete recurrence (default here, NOT the reference's algorithm):
   *     adds the term, mirroring the right side's alpha_last*mu term
   *     (gkl.cpp:155-160); anchored to dense LAPACK SVDs. DESIGN.md section 5. */
  int omega_recurrence;
} gkb_gkl_options;

/* SvdlResult + SvdlStats (gkl.hpp:170-189). Arrays owned by the result. */
typedef struct {
  int64_t m, n, count;  /* count = min(k, steps) */
  double* singvals;     /* count, descending */
  double* U;            /* m x count, column-major */
  double* V;            /* n x count */
  double* err_estimates;/* count */
  int32_t* converged;   /* count */
  int64_t mvps, steps;
  int32_t restarts, reorth_count, deflations, all_converged;
  double wall_seconds;
  int64_t history_len;  /* extractions recorded (record_history) */
  double* ritz_history; /* history_len x k, NaN padded */
  double* err_history;
  /* device-side accounting (not in the reference) */
  double device_seconds;    /* CUDA-event time of the solve on shard 0 */
  int64_t host_syncs;       /* device->host scalar round trips */
  int64_t fused_tails;      /* right half-steps run as one fused cluster launch */
} gkb_svdl_result;

void gkb_gkl_options_default(gkb_gkl_options* o);
/* GklOptions::validate (gkl.cpp:53-73): GKB_EINVAL with the reference message. */
int gkb_gkl_options_validate(const gkb_gkl_options* o, int64_t m, int64_t n);
/* svdl (gkl.hpp:196, gkl.cpp:416-514) with U (SNP side) sharded and V
 * replicated in HBM; the small SVD runs on the host, the per-step decisions
 * (omega recurrences, second passes, breakdown tests) on the device. */
int gkb_svdl(gkb_op* op, const gkb_gkl_options* o, gkb_svdl_result** res);
int gkb_svdl_result_free(gkb_svdl_result* res);

/* SubspaceResult + SubspaceState (subspace.hpp:21-35). Arrays owned by the result. */
typedef struct {
  int64_t m, k;
  double* basis;            /* m x k, column-major */
  double* eigvals;          /* k */
  double* singvals;         /* k */
  int64_t iterations;
  double* delta_history;    /* iterations */
  double* invcond_history;  /* iterations + 1 */
  int32_t converged, rank_deficient;
  int64_t mvps;
} gkb_subspace_result;
/* subspace_iterate (subspace.hpp:50-70, subspace.cpp:49-115), variant kQr,
 * with the k-column blocks resident on the device: gram passes as k + k
 * device products, CholeskyQR2 renormalization (device Gram, k x k host
 * Cholesky), device convergence test. GKB_ELOGIC if the block loses rank
 * (the caller then uses the host-side QR). */
int gkb_subspace_qr(gkb_op* op, int64_t k, double tol, int64_t max_iter, uint64_t seed,
                    int scaled_delta, gkb_subspace_result** res);
int gkb_subspace_result_free(gkb_subspace_result* res);

/* ---- step-level access (LanczosFactorization, gkl.hpp:59-125) ------------
 * For the reference's unit tests of bidiag_step / ritz_extract /
 * thick_restart (proj/tests/test_gkl.cpp). Bases live on the device. */
int gkb_lanczos_create(gkb_op* op, int64_t capacity, const double* start, uint64_t rng_seed,
                       gkb_lanczos** lz);
int gkb_lanczos_destroy(gkb_lanczos* lz);
/* bidiag_step (gkl.cpp:206-312). status: 0 ok, 1 breakdown alpha, 2 breakdown beta. */
int gkb_bidiag_step(gkb_lanczos* lz, const gkb_gkl_options* o, double norm_scale, int* status,
                    int* reorth_left, int* reorth_right, double* alpha, double* beta);
/* steps, capacity, right_exhausted */
int gkb_lanczos_info(gkb_lanczos* lz, int64_t* steps, int64_t* capacity, int* right_exhausted);
/* Downloads U (m x steps), V (n x (steps+1)), B (steps x steps), coupling
 * (steps), omega_left (steps), omega_right (steps+1); NULL skips a field. */
int gkb_lanczos_get(gkb_lanczos* lz, double* U, double* V, double* B, double* coupling,
                    double* omega_left, double* omega_right);
/* ritz_extract (gkl.cpp:314-339): values, W_L, W_R (j x j), err, err_crude, converged */
int gkb_ritz_extract(gkb_lanczos* lz, double tol, double* values, double* WL, double* WR,
                     double* err, double* err_crude, int32_t* converged);
int gkb_thick_restart(gkb_lanczos* lz, int64_t keep);     /* gkl.cpp:341-378 */
int gkb_compress_exhausted(gkb_lanczos* lz);              /* gkl.cpp:380-409 */
/* deflate_right (gkl.cpp:178-204): a fresh right vector drawn from the
 * factorization's Rng (seeded at gkb_lanczos_create) and orthogonalized
 * against V by cgs2, up to 4 attempts; else the right side is exhausted. */
int gkb_deflate_right(gkb_lanczos* lz);

/* ---- primitives -------------------------------------------------------- */
/* cgs2 (orth.hpp:19-44) run on the device: basis len x ncols (host, column-
 * major) is uploaded, v orthogonalized in place, coeffs += basis^T v. */
int gkb_cgs2(gkb_ctx* ctx, const double* basis, int64_t len, int64_t ncols, double* v,
             double* coeffs, double* norm_after);
/* svd_small (small_svd.cpp:14-28), host one-sided Jacobi: M r x c
 * column-major; U r x k, s k, V c x k, k = min(r, c). */
int gkb_svd_small(const double* M, int64_t r, int64_t c, double* U, double* s, double* V);
/* Rng (rng.hpp:17-62): out[i] = uniform_symmetric() for i < n. */
/* Rng(seed).normal() x n (Box-Muller, rng.hpp:46-60). */
int gkb_rng_fill_normal(uint64_t seed, int64_t n, double* out);
int gkb_rng_fill_symmetric(uint64_t seed, int64_t n, double* out);
/* Marker scaling from counts with the reference formulas (see
 * gkb_geno_standardize); exposed for bit-exact checks against the oracle. */
int gkb_marker_scaling(const int64_t* counts, int64_t p, int64_t n, int scheme, double* mu,
                       double* inv_s);

#ifdef __cplusplus
}
#endif
#endif /* GKB_H */
