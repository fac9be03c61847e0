// Launchers for the sm_100a kernels (geno_kernels.cu, basis_kernels.cu,
// synth_kernels.cu). All launches are stream-ordered; no launcher
// synchronizes. Every reduction is fixed-order (block partials summed in
// block order), so results are bitwise reproducible run to run.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace gkb {
namespace dev {

// ---- packed genotype operator -------------------------------------------
// Device layout: the matrix of 2-bit dosage codes r
// (0,1,2 = dosage, 3 = missing, pads 0) is stored twice, as tile layouts:
//   layout 1 (K1 = apply):   rows = local SNPs (p_loc), cols = samples (n)
//   layout 2 (K2 = adjoint): rows = samples (n),       cols = local SNPs
// A tile is 16 rows x 128 cols (8 words of 16 two-bit fields) = 512 B in
// mma.sync fragment order; tiles are stored strip-major (a warp streams one
// 16-row strip along K contiguously).
struct PMPlan {
  int64_t R, C;      // valid rows / cols
  int64_t S;         // 16-row strips, padded to whole CTAs (16 strips = 256 rows)
  int64_t KT;        // 128-col K tiles
  int kt_cta;        // K tiles per CTA column range (2048 cols)
  int nkc;           // column ranges
  int64_t grid_x;    // CTAs along rows (S / strips per CTA)
  int rows_cta;      // rows per CTA (= rows per missing-list block)
  int64_t rows_pad;  // S * 16
  size_t smem;       // main kernel dynamic shared memory (digits)
  size_t dig_smem;   // digitize kernel dynamic shared memory
};
PMPlan pm_plan(int64_t R, int64_t C);
int64_t pm_words(const PMPlan& pl);  // 32-bit words of one layout

// Per-CTA missing lists of one layout (null off when the shard has none):
// block b = kc * grid_x + bx, row r (0..255) owns
//   ent[base[b] + off[b*257 + r] .. base[b] + off[b*257 + r + 1])  (column offsets in the range)
struct MissLists {
  const uint32_t* off;
  const int64_t* base;
  const uint16_t* ent;
};
// Per-product scratch of one layout.
struct PMScratch {
  uint4* dig;     // nkc * kt_cta * 64 B-fragment digits
  int* dexp;      // nkc
  double* dsum;   // nkc
  double* cm;     // K2: c_j (3 - mu_j) per local SNP
  double* part;   // nkc * rows_pad partials
  unsigned* tick; // grid_x arrival counters of the fused K1 finish (zero between launches)
};
struct GenoView {
  const uint4* lt1;
  const uint4* lt2;
  PMPlan pl1, pl2;
  int64_t p_loc, n;
  const double* mu;     // >= pl1.rows_pad (zero beyond p_loc)
  const double* mean;   // observed mean per SNP (imputed value of a missing entry), >= rows_pad
  const double* inv_s;  // >= pl1.rows_pad
  MissLists m1, m2;
  PMScratch s1, s2;
  int64_t nmissing;
  // dense-missing mode (no lists; indicator MMAs, k_pm_ind): s2m holds the
  // digits of K2's cm_j = c_j (3 - m_j)
  bool ind = false;
  PMScratch s2m{};
  // single-layout mode (no layout 2; K2 read from layout 1 by k_pm_adj_l1):
  // blocks of 1024 samples x 1792 SNPs; m2 / s2 are sized for this geometry
  bool single = false;
  int64_t l1t_grid = 0, l1t_nkc = 0, l1t_rows_pad = 0;
};
// tcgen05 block products (k_pm_blk_tc): digits of up to kmax vectors in the
// tcgen05 B-image layout, exponents / sums per (vector, range), partials.
struct TcScratch {
  int kmax = 0;
  uint8_t* dig = nullptr;   // nkc * kt_cta tiles x (8 kmax) rows x 128 B
  uint8_t* dig2 = nullptr;  // K2: digits of cm
  int* dexp = nullptr;      // kmax * nkc
  int* dexp2 = nullptr;
  double* dsum = nullptr;   // kmax * nkc
  double* part = nullptr;   // kmax * nkc * rows_pad
};
// Y[:, v] = X_loc X[:, v] (K1) / Z[:, v] = X_loc^T Y[:, v] (K2, local partial
// sums) for v < k <= 16, one pass over the layout.
void k1_apply_tc(const GenoView& g, const TcScratch& t, const double* X, int64_t ldx, int k,
                 double* Y, int64_t ldy, cudaStream_t s);
void k2_adjoint_tc(const GenoView& g, const TcScratch& t, const double* Yin, int64_t ldy, int k,
                   double* Z, int64_t ldz, cudaStream_t s);
size_t tc_dig_bytes(const PMPlan& pl, int kmax);
int tc_nkc(const PMPlan& pl);  // tcgen05 spans (56 tiles) of a layout

// single-layout K2 geometry of a shard (p_loc SNPs x n samples)
struct L1TPlan {
  int64_t grid_x, nkc, rows_pad;
};
L1TPlan l1t_plan(const PMPlan& pl1, int64_t p_loc);
void miss_lists_l1t(const uint32_t* lay1, const PMPlan& pl1, const L1TPlan& lt, int64_t p_loc,
                    int64_t n, bool fill, uint32_t* cnt, const uint32_t* off, const int64_t* base,
                    uint16_t* ent, cudaStream_t s);
void block_scan_1024(const uint32_t* cnt, int64_t nblk, uint32_t* off, int64_t* tot,
                     cudaStream_t s);
size_t l1t_dig_bytes();  // digits per range

// K8: .bed records of a staging block (rows [row0, row0+rows) of the shard) -> layouts.
void build_lt1(const uint8_t* bed, int64_t stride_bytes, int64_t rows, int64_t row0, int64_t n,
               const PMPlan& pl1, uint32_t* lay1, cudaStream_t s);
void build_lt2(const uint8_t* bed, int64_t stride_bytes, int64_t rows, int64_t row0, int64_t n,
               const PMPlan& pl2, uint32_t* lay2, cudaStream_t s);  // row0 % 16 == 0
// K7: per-SNP [n0, n1, n2, nmiss] from layout 1.
void marker_counts(const uint32_t* lay1, const PMPlan& pl1, int64_t p_loc, int64_t n,
                   int64_t* counts, cudaStream_t s);
// layout 1 -> .bed records for rows [row0, row0+nrows) (read-back check).
void layout_to_bed(const uint32_t* lay1, const PMPlan& pl1, int64_t n, int64_t row0,
                   int64_t nrows, uint8_t* out, cudaStream_t s);
// Missing lists: count pass (fill = false, cnt[nblk*256]), block_scan
// (cnt -> off[nblk*257], tot[nblk]), then the fill pass (needs off and base =
// exclusive scan of tot).
void miss_lists(const uint32_t* lay, const PMPlan& pl, bool fill, uint32_t* cnt,
                const uint32_t* off, const int64_t* base, uint16_t* ent, cudaStream_t s);
void block_scan(const uint32_t* cnt, int64_t nblk, int span, uint32_t* off, int64_t* tot,
                cudaStream_t s);

// K1 apply (reference X*x, per-SNP dot): y (p_loc) = inv_s*(sum r x - mu X_tot - (3-mu) S_miss)
// stream_out: y is written by the main kernel's last CTA of each row block (for
// a page-locked host y: the rows cross PCIe while other blocks still stream);
// otherwise by a separate fixed-order reduce (faster when y stays on the device).
// di.div: the input is x / *di.div (the Lanczos normalization), divided inside
// k_digitize and stored to di.store unless *di.gate == 0 -- what div_copy_dv
// followed by the product does, bit for bit, one launch fewer.
struct DivIn {
  const double* div = nullptr;
  double* store = nullptr;
  const int* gate = nullptr;
};
void k1_apply(const GenoView& g, const double* x, double* y, cudaStream_t s,
              bool stream_out = false, const DivIn& di = DivIn());
// K2 apply_adjoint (reference X^T*y, per-sample sum) over the local SNPs; z has n entries.
void k2_adjoint(const GenoView& g, const double* y, double* z, cudaStream_t s,
                const DivIn& di = DivIn());
// Two vectors per pass (block products): each column bitwise equal to the
// single-vector product. `sb` is a second scratch set of the layout (vector 1).
void k1_apply2(const GenoView& g, const PMScratch& sb, const double* x0, const double* x1,
               double* y0, double* y1, cudaStream_t s);
void k2_adjoint2(const GenoView& g, const PMScratch& sb, const double* y0, const double* y1,
                 double* z0, double* z1, cudaStream_t s);
// Per-marker fits y ~ [1, m_i, Z] from the block product P = X [y, C] (rows x
// (K+1), ldp) and the shared nuisance algebra (K = columns of C = [1, Z]).
void marker_scan(const GenoView& g, const double* P, int64_t ldp, int K, const double* Ainv,
                 const double* w, double yyc, double a0w, double denom, const int64_t* counts,
                 double* beta, double* se, double* icpt, double* sig2, int* dep, cudaStream_t s);
// Pieces (for timing breakdowns): digitize, then the main tensor-core kernel.
void k1_digitize(const GenoView& g, const double* x, cudaStream_t s, const DivIn& di = DivIn());
void k2_digitize(const GenoView& g, const double* y, cudaStream_t s, const DivIn& di = DivIn());
void k1_main_only(const GenoView& g, const double* x, cudaStream_t s);
void k2_main_only(const GenoView& g, cudaStream_t s);

// ---- dense fp64 basis / operator kernels (K3-K6) -------------------------
// Reduction scratch: per-CTA partials and the last-CTA ticket of the
// single-launch reductions (one reduction in flight per stream).
namespace ctl {
struct Post;  // a light step decision run by the reduction's last CTA (below)
}
struct RedScratch {
  double* partial;
  int64_t cap;  // doubles
  unsigned* ticket = nullptr;
};
int64_t red_blocks(int64_t len);  // CTAs of a reduction over len rows (partials per column)
void init_red_scratch(RedScratch& rs);  // allocates the zeroed ticket

// out[0..ncols) = Q[:, c0:c0+ncols]^T v ; out[ncols] = ||v||^2 (if with_norm)
void gemv_t(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* v, bool with_norm,
            RedScratch& rs, double* out, cudaStream_t s, const int* gate = nullptr);
// v = beta*v - Q c (c on device, ncols) ; if norms: out[0] = ||v_before||^2, out[1] = ||v_after||^2
// (beta applies to v before the subtraction; used for dense apply with beta = 0 -> y = -Qc).
void gemv_n(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* c, double* v,
            double beta, double sign, bool norms, RedScratch& rs, double* out, cudaStream_t s,
            const int* gate = nullptr, const ctl::Post* post = nullptr);
// out[0] = sum a*b ; (dot into device scalar)
void dot(const double* a, const double* b, int64_t len, RedScratch& rs, double* out, cudaStream_t s,
         const int* gate = nullptr, const ctl::Post* post = nullptr);
// out[0] = ||a||^2
void nrm2sq(const double* a, int64_t len, RedScratch& rs, double* out, cudaStream_t s,
            const int* gate = nullptr, const ctl::Post* post = nullptr);
// v -= (*dprev) * uprev (if uprev and agate on), then out[0] = sum unext * v
// (||v||^2 when unext is null) if dgate on: axpy_dev + dot in one pass, same bits.
void axpy_dot(const double* dprev, const double* uprev, const int* agate, const double* unext,
              const int* dgate, double* v, int64_t len, RedScratch& rs, double* out,
              cudaStream_t s);
// out[0] = sum (a - b)^2
void diff_nrm2sq(const double* a, const double* b, int64_t len, RedScratch& rs, double* out,
                 cudaStream_t s);
// v -= (*dptr) * u   (device scalar)
void axpy_dev(const double* dptr, const double* u, double* v, int64_t len, cudaStream_t s,
              const int* gate = nullptr);
// v = v - alpha*u, with out[0] = ||v_before||^2, out[1] = ||v_after||^2
void axpy_norms(double alpha, const double* u, double* v, int64_t len, RedScratch& rs, double* out,
                cudaStream_t s);
// dst = src / divisor (the reference divides: w /= alpha, gkl.cpp:253)
void div_copy(const double* src, double divisor, double* dst, int64_t len, cudaStream_t s);
// Same two operations with the scalar taken as sqrt(*nrm2) on the device
// (bitwise equal to the host's sqrt of the same value): lets the driver launch
// the next half-step before the host has read the norm.
void div_copy_dsq(const double* src, const double* nrm2, double* dst, int64_t len, cudaStream_t s);
void axpy_norms_dsq(const double* nrm2, const double* u, double* v, int64_t len, RedScratch& rs,
                    double* out, cudaStream_t s);
// Device-scalar variants for the device-controlled step (scalar = *alpha /
// *divisor, no sqrt), gated: nothing happens when *gate == 0. Every kernel
// above that takes a `gate` behaves the same way.
void axpy_norms_dv(const double* alpha, const double* u, double* v, int64_t len, RedScratch& rs,
                   double* out, cudaStream_t s, const int* gate, const ctl::Post* post = nullptr);
void div_copy_dv(const double* src, const double* divisor, double* dst, int64_t len,
                 cudaStream_t s, const int* gate);
// dst[:, 0:kc] = Q[:, 0:j] * W (W is j x kc, ldw rows, on device); dst may not alias Q
void gemm_small(const double* Q, int64_t ld, int64_t len, int64_t j, const double* W, int64_t ldw,
                int64_t kc, double* dst, int64_t ldd, cudaStream_t s);
// dst = sum_k srcs[k] (k in order), nsrc <= 16
void sum_buffers(const double* const* srcs, int nsrc, double* dst, int64_t len, cudaStream_t s);
// L2 flush: write `bytes` of scratch
void flush_l2(void* buf, size_t bytes, cudaStream_t s);

// ---- device-side step control (ctl_kernels.cu) ----------------------------
// Per shard: one double area (B, couplings, omega rows, scalars, reduction
// results) and one int area (gates, status, counters), identical replicas on
// every shard. Gates are read by the gated kernels above.
namespace ctl {
enum : int {  // int slots
  I_ALIVE = 0,   // 0 after a breakdown: every later gated kernel does nothing
  I_STATUS,      // 0, or the StepInfo status of the step that halted the run
  I_J,           // factorization size
  I_STEPS,       // completed steps (status 0 or 2)
  I_REORTH,      // partial-mode reorthogonalizations (both sides)
  I_G2P,         // local second pass on
  I_GRE,         // reorthogonalize (cgs2 pass 1) on
  I_GRE2,        // cgs2 second pass on
  I_RPEND,       // reorthogonalizations of the current step (committed with the step)
  I_G2PC         // + c: second-pass term c on (cap entries)
};
enum : int { S_NS = 0, S_ALPHA, S_BETA, S_ACAND, S_BCAND, S_NAFTER, S_COUNT = 16 };  // scalars
enum : int { R_N = 0, R_DOT = 8, R_CG = 16 };  // result slots: norm pair, dot, cgs2 coefficients
struct Layout {  // offsets in doubles
  int64_t cap, B, coup, mu, nu, mun, nun, sc, res, nd, ni;
  size_t bytes;
};
__host__ __device__ inline Layout layout(int64_t cap) {
  Layout L;
  L.cap = cap;
  L.B = 0;
  L.coup = L.B + cap * cap;
  L.mu = L.coup + cap;
  L.nu = L.mu + cap + 2;
  L.mun = L.nu + cap + 1;
  L.nun = L.mun + cap + 2;
  L.sc = L.nun + cap + 1;
  L.res = L.sc + S_COUNT;
  L.nd = L.res + 3 * cap + 32;
  L.ni = I_G2PC + cap;
  L.bytes = sizeof(double) * (size_t)L.nd + sizeof(int) * (size_t)L.ni;
  return L;
}
enum Op { OP_L_A, OP_L_B, OP_CG_MID, OP_CG_END, OP_L_END, OP_R_A, OP_R_B, OP_R_END, OP_SQRT_L };
struct Params {
  int op, side, full, nidx, has_pattern, omega_rec, one_sided;
  int then_op;  // a second decision in the same launch (-1: none)
  int64_t s, ncols, lo, hi, m, n, cap;
  double omega, lvl, bfac, guard, eta, eps;
};
void launch(double* d, int* iv, const Params& p, cudaStream_t st);
// The right half-step after the adjoint's reduction, fused (ctl_kernels.cu
// k_right_tail): partial mode's axpy + norms, R_A, local second pass, R_B,
// then cgs2 (gated) with CG_MID / CG_END and R_END -- one cluster launch for
// n <= kTailMaxN, the unfused kernels' bits. V: n x (s + 1), ld n. Returns
// false (nothing enqueued) when it does not apply; the caller then enqueues
// the unfused sequence.
constexpr int64_t kTailMaxN = 16 * 256 * 4;
struct TailArgs {
  double* d;
  int* iv;
  Params p;  // ctl_params(o, OP_R_B, s)
  const double* V;
  double* z;
  int64_t n;
  unsigned long long* tlog = nullptr;  // GKB_RTAIL_TLOG: per-phase SM cycles of CTA 0 (debug)
};
bool right_tail(const TailArgs& a, cudaStream_t st);
// A light decision (OP_L_A, OP_R_A, OP_CG_MID: ctl_ops.cuh) handed to the
// reduction that produces its inputs: its last CTA runs it after the finalize
// (block 0 when the reduction is gated off), saving the ctl launch. Only where
// no allreduce sits between the two (right side, or one shard in total).
struct Post {
  double* d = nullptr;
  int* iv = nullptr;
  Params p{};
};
}  // namespace ctl

// ---- synthetic generator ------------------------------------------------
struct SynthDev {
  int64_t p, n;
  uint64_t seed;
  int npop;
  const double* freq;       // npop x p (device)
  const int32_t* pop;       // n or null
  const double* admix;      // n x npop or null
  double missing_rate;
  const int32_t* copy_from; // n or null
  double copy_prob;
};
// Writes .bed records for markers [j0, j0+rows) into out (stride ceil(n/4)).
void synth_bed(const SynthDev& sp, int64_t j0, int64_t rows, uint8_t* out, cudaStream_t s);

}  // namespace dev
}  // namespace gkb
