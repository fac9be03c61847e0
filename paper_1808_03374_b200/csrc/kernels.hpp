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
// Device layout: the p_loc x n matrix of 2-bit dosage
// codes r (0,1,2 = dosage, 3 = missing, pads 0) is cut into 16-byte chunks
// (4 consecutive SNPs x one 32-bit word of 16 samples). Two orderings:
//   layout A ("row-quad", for the adjoint K2): chunk (q, w) at q*W + w
//   layout B ("col-quad", for the apply K1):   chunk (q, w) at w*P4 + q
// W = ceil(n/16) words per SNP, P4 = ceil(p_loc/4) SNP quads.
struct GenoView {
  const uint4* layA;
  const uint4* layB;
  int64_t p_loc, n, W, P4;
  const double* mu;     // p_loc
  const double* inv_s;  // p_loc
  // Per-CTA missing lists (null when the shard has no missing entries):
  // block b, row r owns ent[base[b] + off[b*(span+1)+r] .. base[b] + off[b*(span+1)+r+1]).
  // m1: K1 blocks b = tile*grid_x + qb, span 128 SNP rows, entries = sample offset in the tile
  // m2: K2 blocks b = chunk*grid_x + wb, span 512 samples, entries = SNP offset in the chunk
  const uint32_t* m1_off;
  const int64_t* m1_base;
  const uint16_t* m1_ent;
  const uint32_t* m2_off;
  const int64_t* m2_base;
  const uint16_t* m2_ent;
  int64_t nmissing;
};

// K8: .bed records [rows of one staging block] -> both layouts.
void build_layouts(const uint8_t* bed, int64_t stride_bytes, int64_t rows_in_block, int64_t q_base,
                   int64_t n, int64_t W, int64_t P4, uint4* layA, uint4* layB, cudaStream_t s);
// K7: per-SNP [n0, n1, n2, nmiss] from layout A.
void marker_counts(const uint4* layA, int64_t P4, int64_t W, int64_t p_loc, int64_t n,
                   int64_t* counts, cudaStream_t s);
// layout A -> .bed records for rows [row0, row0+nrows) (read-back check).
void layout_to_bed(const uint4* layA, int64_t P4, int64_t W, int64_t n, int64_t row0,
                   int64_t nrows, uint8_t* out, cudaStream_t s);

struct K1Plan {
  int tileW;     // 32-bit words (16 samples) per sample tile
  int ntiles;
  int64_t grid_x;
  size_t smem;
};
K1Plan k1_plan(int64_t W, int64_t P4);
// K1 apply (reference X*x, per-SNP dot): y (p_loc) = inv_s*(sum r x - mu X_tot - (3-mu) S_miss)
// scratch: ypart ntiles*4*P4 doubles.
void k1_apply(const GenoView& g, const K1Plan& pl, const double* x, double* ypart, double* y,
              cudaStream_t s);

struct K2Plan {
  int qc;        // SNP quads per chunk
  int nchunks;
  int64_t grid_x;
  size_t smem;
  int minb;      // __launch_bounds__ min blocks of the k2_main instance (3 or 4)
};
K2Plan k2_plan(int64_t W, int64_t P4);
// K2 apply_adjoint (reference X^T*y, per-sample sum) over the local SNPs.
// scratch: zpart nchunks*16*W doubles. z has n entries.
void k2_adjoint(const GenoView& g, const K2Plan& pl, const double* y, double* zpart, double* z,
                cudaStream_t s);
// The two main packed kernels alone (for timing breakdowns).
void k1_main_only(const GenoView& g, const K1Plan& pl, const double* x, double* ypart,
                  cudaStream_t s);
void k2_main_only(const GenoView& g, const K2Plan& pl, const double* y, double* zpart,
                  cudaStream_t s);

// Per-CTA missing lists for the two plans: count pass (fill = false, writes
// cnt[nblk*span]), block_scan (cnt -> off[nblk*(span+1)], tot[nblk]), then the
// fill pass (fill = true, needs off and base = exclusive scan of tot).
void miss_lists_k1(const uint4* layA, int64_t P4, int64_t W, const K1Plan& pl, bool fill,
                   uint32_t* cnt, const uint32_t* off, const int64_t* base, uint16_t* ent,
                   cudaStream_t s);
void miss_lists_k2(const uint4* layA, int64_t P4, int64_t W, const K2Plan& pl, bool fill,
                   uint32_t* cnt, const uint32_t* off, const int64_t* base, uint16_t* ent,
                   cudaStream_t s);
void block_scan(const uint32_t* cnt, int64_t nblk, int span, uint32_t* off, int64_t* tot,
                cudaStream_t s);

// ---- dense fp64 basis / operator kernels (K3-K6) -------------------------
// Reduction scratch: partial[nblk * K] plus the result buffer.
struct RedScratch {
  double* partial;
  int64_t cap;  // doubles
};
int64_t red_blocks(int64_t len);

// out[0..ncols) = Q[:, c0:c0+ncols]^T v ; out[ncols] = ||v||^2 (if with_norm)
void gemv_t(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* v, bool with_norm,
            RedScratch& rs, double* out, cudaStream_t s);
// v = beta*v - Q c (c on device, ncols) ; if norms: out[0] = ||v_before||^2, out[1] = ||v_after||^2
// (beta applies to v before the subtraction; used for dense apply with beta = 0 -> y = -Qc).
void gemv_n(const double* Q, int64_t ld, int64_t len, int64_t ncols, const double* c, double* v,
            double beta, double sign, bool norms, RedScratch& rs, double* out, cudaStream_t s);
// out[0] = sum a*b ; (dot into device scalar)
void dot(const double* a, const double* b, int64_t len, RedScratch& rs, double* out, cudaStream_t s);
// out[0] = ||a||^2
void nrm2sq(const double* a, int64_t len, RedScratch& rs, double* out, cudaStream_t s);
// v -= (*dptr) * u   (device scalar)
void axpy_dev(const double* dptr, const double* u, double* v, int64_t len, cudaStream_t s);
// v = v - alpha*u, with out[0] = ||v_before||^2, out[1] = ||v_after||^2
void axpy_norms(double alpha, const double* u, double* v, int64_t len, RedScratch& rs, double* out,
                cudaStream_t s);
// dst = src / divisor (the reference divides: w /= alpha, gkl.cpp:253)
void div_copy(const double* src, double divisor, double* dst, int64_t len, cudaStream_t s);
// dst[:, 0:kc] = Q[:, 0:j] * W (W is j x kc, ldw rows, on device); dst may not alias Q
void gemm_small(const double* Q, int64_t ld, int64_t len, int64_t j, const double* W, int64_t ldw,
                int64_t kc, double* dst, int64_t ldd, cudaStream_t s);
// dst = sum_k srcs[k] (k in order), nsrc <= 16
void sum_buffers(const double* const* srcs, int nsrc, double* dst, int64_t len, cudaStream_t s);
// L2 flush: write `bytes` of scratch
void flush_l2(void* buf, size_t bytes, cudaStream_t s);

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
