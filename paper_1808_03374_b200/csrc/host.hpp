// Host-side structures of the B200 GKL library: context (shards, streams,
// communicator), device operators (packed genotype, dense) and the GKL
// driver with device-resident Krylov bases.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <memory>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "gkb_common.hpp"
#include "kernels.hpp"

namespace gkb {

// RAII holders for scratch allocations on error paths (a GKB_CUDA throw
// inside guarded() must not leak device memory or events).
struct DevScratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;  // non-null: stream-ordered (cudaFreeAsync)
  DevScratch() = default;
  DevScratch(const DevScratch&) = delete;
  DevScratch& operator=(const DevScratch&) = delete;
  ~DevScratch() {
    if (p) {
      if (st) cudaFreeAsync(p, st);
      else cudaFree(p);
    }
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};
struct PinnedScratch {  // cudaMallocHost'd staging buffer
  void* p = nullptr;
  PinnedScratch() = default;
  PinnedScratch(const PinnedScratch&) = delete;
  PinnedScratch& operator=(const PinnedScratch&) = delete;
  ~PinnedScratch() {
    if (p) cudaFreeHost(p);
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};
struct EventHolder {
  cudaEvent_t e = nullptr;
  EventHolder() = default;
  EventHolder(const EventHolder&) = delete;
  EventHolder& operator=(const EventHolder&) = delete;
  ~EventHolder() {
    if (e) cudaEventDestroy(e);
  }
};

// Rng (rng.hpp:17-62): std::mt19937_64 with the reference's draw algorithms.
class Rng {
 public:
  explicit Rng(uint64_t seed) : engine_(seed) {}
  uint64_t bits() { return engine_(); }
  double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  double uniform_symmetric() { return 2.0 * uniform() - 1.0; }
  // Box-Muller; one engine pair feeds two variates (rng.hpp:46-60, bit-exact:
  // same draws, same libm calls)
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    constexpr double two_pi = 6.283185307179586476925286766559;
    spare_ = radius * std::sin(two_pi * u2);
    have_spare_ = true;
    return radius * std::cos(two_pi * u2);
  }

 private:
  std::mt19937_64 engine_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

// One SNP shard: a device, a stream, scratch for fixed-order reductions and
// pinned staging for scalar read-backs.
struct Shard {
  int index = 0;  // global shard index (rank in SPMD mode)
  int dev = 0;
  cudaStream_t stream = nullptr;
  dev::RedScratch rs{nullptr, 0};
  double* dres = nullptr;  // device results (res_cap doubles, >= kResCap)
  double* hres = nullptr;  // pinned host mirror
  int64_t res_cap = 0;
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  cudaEvent_t ev = nullptr;
  void ensure_partial(int64_t doubles);
  // grow dres / hres to hold `doubles` results (synchronizes the stream when it
  // reallocates; callers must re-read s.dres / s.hres afterwards)
  void ensure_res(int64_t doubles);
  // pinned host staging for file ingest (two buffers, grow-only, kept)
  uint8_t* hstage[2] = {nullptr, nullptr};
  size_t hstage_bytes = 0;
  uint8_t* pinned_stage(int k, size_t bytes);
};

constexpr int64_t kResCap = 1 << 16;
// device -> pageable host copy through the shard's page-locked staging (synchronous)
void d2h_staged(Shard& s, void* dst, const void* src, size_t bytes);

struct Context {
  std::vector<Shard> shards;
  int nshards_total = 1;
  int first_shard = 0;
  // SPMD: one shard per process, collectives across processes -- over NCCL
  // (gkb_init_nccl), or through a caller-supplied host allreduce
  // (gkb_init_host_comm: stream-ordered D2H -> host function -> H2D, used to
  // run the SPMD path as several processes on one GPU, e.g. over gloo)
  bool spmd_mode = false;
  ncclComm_t comm = nullptr;
  gkb_host_allreduce_fn host_fn = nullptr;
  void* host_user = nullptr;
  double* host_buf = nullptr;  // page-locked staging of the host allreduce
  int64_t host_cap = 0;
  // local-mode allreduce staging on shard 0's device
  double* stage = nullptr;
  int64_t stage_cap = 0;

  ~Context();
  void init_local(const std::vector<int>& devices);
  void init_nccl(int device, const ncclUniqueId& id, int nranks, int rank);
  void init_host(int device, int nranks, int rank, gkb_host_allreduce_fn fn, void* user);
  // In-place sum over all shards (all processes). bufs: one device pointer per
  // local shard. Result identical on every shard.
  void allreduce(const std::vector<double*>& bufs, int64_t count);
  void sync_all();
  void set_device(int i) const;
};

// Contiguous row partition; interior boundaries multiples of 4.
std::vector<int64_t> partition_rows(int64_t m, int nparts);

// Device linear operator (LinearOperator, linop.hpp:13-39) with rows
// (reference m = SNPs) sharded and columns (samples) replicated.
struct DevOp {
  Context* ctx = nullptr;
  int64_t m = 0, n = 0;
  std::vector<int64_t> starts;  // global partition, nshards_total + 1
  int64_t mvps = 0;
  // host-API staging buffers per local shard
  std::vector<double*> xbuf, ybuf, zbuf, yfull;
  // the operator's kernels may read the adjoint input and write the results
  // straight from/to page-locked host buffers (each element touched once)
  bool direct_host_io = false;
  bool host_out_ = false;  // set by apply_host while its result buffer is page-locked host memory

  virtual ~DevOp();
  int64_t row0(int i) const { return starts[ctx->shards[i].index]; }
  int64_t rows(int i) const { return starts[ctx->shards[i].index + 1] - starts[ctx->shards[i].index]; }
  // y_i (rows(i)) = X_i x_i ; x_i replicated (n). Stream-ordered on shard streams.
  virtual void apply_dev(const std::vector<const double*>& x, const std::vector<double*>& y) = 0;
  // z (n) = sum_i X_i^T y_i, allreduced so every shard holds the full z.
  virtual void adjoint_dev(const std::vector<const double*>& y, const std::vector<double*>& z) = 0;
  // The same products of x_raw / *div[i], the quotient stored to xs[i] unless
  // *gate[i] == 0 (the Lanczos normalization before each product). Default:
  // div_copy_dv, then the product; the genotype operator divides while it
  // digitizes the input (one launch fewer, same bits).
  virtual void apply_dev_div(const std::vector<const double*>& xraw,
                             const std::vector<const double*>& div,
                             const std::vector<const int*>& gate, const std::vector<double*>& xs,
                             const std::vector<double*>& y);
  virtual void adjoint_dev_div(const std::vector<const double*>& yraw,
                               const std::vector<const double*>& div,
                               const std::vector<const int*>& gate, const std::vector<double*>& ys,
                               const std::vector<double*>& z);
  void alloc_host_api_buffers();
  void apply_host(const double* x, double* y);
  void adjoint_host(const double* y, double* z);
  bool direct_io(const void* a, const void* b) const;
  // k columns per call (column-major host blocks): one H2D, k device products
  // back to back, one D2H (the block form subspace iteration uses)
  // Device blocks, column-major per shard: X[i] n x k (ldx), Y[i] rows(i) x k
  // (ldy[i]); the adjoint's Z[i] n x k (ldz) is summed across shards. Default:
  // one column at a time; an operator may do several columns per pass.
  virtual void apply_block_dev(const std::vector<const double*>& X, int64_t ldx, int64_t k,
                               const std::vector<double*>& Y, const std::vector<int64_t>& ldy);
  virtual void adjoint_block_dev(const std::vector<const double*>& Yb,
                                 const std::vector<int64_t>& ldyb, int64_t k,
                                 const std::vector<double*>& Z, int64_t ldz);
  void apply_block_host(const double* X, int64_t k, double* Y);
  void adjoint_block_host(const double* Y, int64_t k, double* Z);
  std::vector<double*> bin_, bout_;  // per shard block buffers (grow-only)
  int64_t bin_cap_ = 0, bout_cap_ = 0;
  void ensure_block_buffers(int64_t in_doubles, int64_t out_doubles);
};

// read_bed's checks (genio.cpp:53-70) on the three files; fills p, n.
void bed_check(const char* bed, const char* bim, const char* fam, int64_t* p, int64_t* n);

struct GenoShard {
  int64_t p_loc = 0, n = 0;
  dev::PMPlan pl1{}, pl2{};   // layout 1 (rows SNPs) / layout 2 (rows samples)
  uint32_t* lt1 = nullptr;
  uint32_t* lt2 = nullptr;
  double* mu = nullptr;       // pl1.rows_pad entries, zero beyond p_loc
  double* mean = nullptr;     // observed means (impute_mean's value), pl1.rows_pad entries
  double* inv_s = nullptr;
  int64_t* counts = nullptr;  // device p_loc*4
  int64_t nmissing = 0;
  dev::PMScratch s1b{}, s2b{};  // second scratch sets (two-vector block products), lazily
  // per-CTA missing lists of the two layouts (kernels.hpp MissLists)
  uint32_t* m1_off = nullptr;
  int64_t* m1_base = nullptr;
  uint16_t* m1_ent = nullptr;
  uint32_t* m2_off = nullptr;
  int64_t* m2_base = nullptr;
  uint16_t* m2_ent = nullptr;
  int64_t list_bytes = 0;
  dev::PMScratch s1{}, s2{};
  // dense-missing mode (kernels.hpp GenoView::ind): chosen at build from the
  // shard's missing fraction (GKB_MISS_MODE=list|ind|auto)
  bool ind = false;
  dev::PMScratch s2m{};
  // single-layout mode (kernels.hpp GenoView::single): chosen at allocation
  // by plan_layouts (GKB_LAYOUTS=1|2 forces)
  bool single = false;
  dev::L1TPlan plt{};
  dev::TcScratch tc1{}, tc2{};  // tcgen05 block products (lazily, k_pm_blk_tc)
  dev::GenoView view() const;
};

// Device-memory plan of one shard (p_loc SNPs x n samples): both tile
// layouts when they fit in `free_bytes` (with the lists, scratch and a solver
// headroom), else layout 1 only (K2 by k_pm_adj_l1).
struct LayoutPlan {
  int layouts = 2;
  int64_t dual_bytes = 0, single_bytes = 0;
};
LayoutPlan plan_layouts(int64_t p_loc, int64_t n, double missing_fraction, int64_t free_bytes);

struct GenoOp : DevOp {
  GenoOp() { direct_host_io = true; }  // k1_reduce writes y, k_digitize<1> reads y, k2_reduce writes z
  std::vector<GenoShard> gs;
  std::vector<int64_t> counts_host;  // p*4 (local rows only in SPMD mode, zero elsewhere)
  bool scaled = false;
  double plan_missing = 0.02;  // missing fraction assumed by the layout plan (synth: the spec's)
  ~GenoOp() override;
  void build_from_payload(const uint8_t* payload, int64_t p, int64_t n);
  void build_from_bed_file(const char* bed, int64_t p, int64_t n);  // after bed_check
  void build_from_synth(const dev::SynthDev& spec_host_ptrs, const gkb_synth_spec* spec);
  void finish_build();  // counts, missing lists, plans, scratch
  void set_scaling(const double* mu, const double* inv_s);  // global p arrays
  void get_scaling(double* mu, double* inv_s);
  void apply_dev(const std::vector<const double*>& x, const std::vector<double*>& y) override;
  void apply_block_dev(const std::vector<const double*>& X, int64_t ldx, int64_t k,
                       const std::vector<double*>& Y, const std::vector<int64_t>& ldy) override;
  void adjoint_block_dev(const std::vector<const double*>& Yb, const std::vector<int64_t>& ldyb,
                         int64_t k, const std::vector<double*>& Z, int64_t ldz) override;
  void adjoint_dev(const std::vector<const double*>& y, const std::vector<double*>& z) override;
  void apply_dev_div(const std::vector<const double*>& xraw, const std::vector<const double*>& div,
                     const std::vector<const int*>& gate, const std::vector<double*>& xs,
                     const std::vector<double*>& y) override;
  void adjoint_dev_div(const std::vector<const double*>& yraw,
                       const std::vector<const double*>& div, const std::vector<const int*>& gate,
                       const std::vector<double*>& ys, const std::vector<double*>& z) override;
  int64_t packed_bytes() const;
  int64_t device_bytes() const;
  // per-marker regression scan (regress.py marker_scan) with the block product
  // and the per-marker algebra on the device; host outputs of length m
  void marker_scan(const double* y, const double* Z, int64_t k, bool unbiased, double* beta,
                   double* se, double* icpt, double* sig2, int32_t* dep);
  void read_bed(int64_t row0, int64_t nrows, uint8_t* out);

 private:
  void alloc_shard(int i, int64_t p_loc, int64_t n);
};

struct DenseOp : DevOp {
  std::vector<double*> X;  // per shard rows(i) x n, ld = rows(i)
  ~DenseOp() override;
  void build(const double* Xh, int64_t m, int64_t n);
  void apply_dev(const std::vector<const double*>& x, const std::vector<double*>& y) override;
  void adjoint_dev(const std::vector<const double*>& y, const std::vector<double*>& z) override;
};

// Marker scaling from counts (genio.cpp:150-185 restated on counts).
void marker_scaling(const int64_t* counts, int64_t p, int64_t n, int scheme, double* mu, double* inv_s);

// svd_small (small_svd.cpp:14-28) -- host one-sided Jacobi.
void svd_small(const double* M, int64_t r, int64_t c, double* U, double* s, double* V);

// ---- GKL (gkl.hpp / gkl.cpp) ----------------------------------------------
struct Options {
  int64_t k = 10;
  double tol = 1e-8;
  int64_t max_mvps = 1000000;
  bool full = false;  // reorth == kFull
  double omega = 1e-8;
  bool one_sided = false;
  bool thick = false;  // restart == kThick
  int64_t max_subspace = 40;
  int64_t keep = 20;
  uint64_t seed = 0;
  bool record_history = false;
  int omega_recurrence = 1;
};
Options options_from(const gkb_gkl_options* o);
void validate_options(const Options& o, int64_t m, int64_t n);  // throws GKB_EINVAL

struct Ritz {
  int64_t j = 0;
  std::vector<double> values, WL, WR, err, err_crude;
  std::vector<int32_t> converged;
};

struct StepInfo {
  int status = 0;  // 0 ok, 1 alpha breakdown, 2 beta breakdown
  bool reorth_left = false, reorth_right = false;
  double alpha = 0.0, beta = 0.0;
};

class Lanczos {
 public:
  Lanczos(DevOp* op, int64_t capacity, const double* start_host, uint64_t rng_seed);
  ~Lanczos();
  int64_t steps() const { return j_; }
  int64_t version() const { return version_; }  // bumped by every change of the factorization
  int64_t capacity() const { return cap_; }
  bool right_exhausted() const { return right_exhausted_; }
  StepInfo step(const Options& o, double norm_scale, int64_t* mvp_counter);
  Ritz ritz_extract(double tol) const;
  // `current`: ritz_extract of the present factorization if the caller has it
  void thick_restart(int64_t keep, const Ritz* current = nullptr);
  void compress_exhausted();
  void deflate_right();
  // downloads (host arrays sized by the caller)
  void get(double* U, double* V, double* B, double* coupling, double* om_left, double* om_right);
  // out_U (m x kc) = U[:, :j] W_L[:, :kc], out_V (n x kc) = V[:, :j] W_R[:, :kc]
  void ritz_vectors(const Ritz& r, int64_t kc, double* outU, double* outV);
  double cgs2_right_host(int64_t ncols);  // test hook
  // Device-controlled steps (ctl_kernels.cu): enqueues up to `nsteps` steps
  // with every decision taken on the device, then one read-back. Stops at the
  // first breakdown (status 1 / 2 as in StepInfo); the host then handles it
  // as after step(). norm_scale is read and updated (svdl's running value).
  struct DevRun {
    int64_t completed = 0;  // steps with status 0 or 2
    int status = 0;
    int64_t reorth = 0;
  };
  DevRun run_dev(const Options& o, int64_t nsteps, double* norm_scale);
  int64_t host_syncs = 0;
  int64_t fused_tails = 0;  // right_tail_dev launches
  unsigned long long* tlog_ = nullptr;  // GKB_RTAIL_TLOG (debug; printed and freed at destruction)
  double t_enqueue = 0.0, t_wait = 0.0;  // run_dev host phases (GKB_VERBOSE)
  int64_t spec_hits = 0, spec_misses = 0;  // speculative right half-steps kept / not launched or redone
  Rng rng;

 private:
  enum Side { kLeft = 0, kRight = 1 };
  DevOp* op_;
  Context* ctx_;
  int64_t m_, n_, cap_, j_ = 0;
  int64_t version_ = 0;
  std::vector<double*> U_, V_, U2_, V2_, w_, z_, cbuf_;
  std::vector<double> B_, coupling_, mu_, nu_, mu_next_, nu_next_;
  bool right_exhausted_ = false;

  double& B(int64_t i, int64_t c) { return B_[i + c * cap_]; }
  double Bc(int64_t i, int64_t c) const { return B_[i + c * cap_]; }
  int64_t len(Side s, int i) const { return s == kLeft ? op_->rows(i) : n_; }
  const std::vector<double*>& basis(Side s) const { return s == kLeft ? U_ : V_; }
  int64_t ld(Side s, int i) const { return s == kLeft ? op_->rows(i) : n_; }
  void read(int64_t count);  // D2H shard-0 dres[0..count) -> hres, sync
  // D2H shard-0 dres[off..off+count) -> hres (same offsets) + event; no sync
  void read_async(int64_t off, int64_t count, cudaEvent_t ev);
  void wait_event(cudaEvent_t ev);  // host waits for a read_async (counts a host sync)
  // u_s = w / alpha, z = X^T u_s, (partial) z -= alpha v_s + norms -> hres[kRightSlot..]
  void launch_right(int64_t s, const std::vector<double*>& dres, int64_t nidx, bool dev_alpha,
                    double alpha, bool partial);
  static constexpr int64_t kRightSlot = 16;  // dres/hres slot of the right half-step norms
  cudaEvent_t ev_left_ = nullptr, ev_right_ = nullptr;
  bool speculate_ = true;  // launch the right half-step before the host reads alpha
  bool left_reorth_unlikely(const Options& o, double norm_scale) const;
  double cgs2(Side side, int64_t ncols, const std::vector<double*>& vec);
  bool partial_reorth_update(Side side, const std::vector<double*>& cand, double cand_coeff,
                             const Options& o, double norm_scale, double* new_norm);
  void upload_small(const std::vector<double>& W, std::vector<double*>& dst);
  std::vector<double*> tmp_small_;
  int64_t tmp_cap_ = 0;
  static constexpr int kRing = 4;  // pinned staging slots for host_to_all
  std::vector<double*> ring_slot_;
  std::vector<cudaEvent_t> ring_ev_;  // kRing x shards
  std::vector<char> ring_used_;
  int64_t ring_cap_ = 0;
  int ring_next_ = 0;
  void host_to_all(const double* h, int64_t count, std::vector<double*>& dst);
  // device step control state (one replica per shard) and pinned staging
  dev::ctl::Layout ctl_L_{};
  std::vector<void*> ctl_d_;
  void* ctl_up_ = nullptr;
  void* ctl_down_ = nullptr;
  double* cd(int i) const { return reinterpret_cast<double*>(ctl_d_[i]); }
  int* ci(int i) const { return reinterpret_cast<int*>(cd(i) + ctl_L_.nd); }
  bool right_tail_dev(const Options& o, int64_t s);
  void enqueue_step_dev(const Options& o, int64_t s, int64_t lo, int64_t hi, bool last);
  bool v_pending_ = false;  // v_{s+1} = z / beta left to the next step's apply (same run)
  void cgs2_dev(Side side, int64_t ncols, const std::vector<double*>& vec, int gate_slot,
                const Options& o, int64_t s, int then_op = -1);
  static bool fuse_ctl();
  bool reduce_local() const;
  dev::ctl::Params ctl_params(const Options& o, int op, int64_t s) const;
};

struct SvdlOutput {
  std::vector<double> singvals, err;
  // Ritz vectors, column-major m x count / n x count (new[]: handed to the C
  // ABI result as they are, no copy or zero fill)
  std::unique_ptr<double[]> U, V;
  std::vector<int32_t> converged;
  int64_t count = 0, mvps = 0, steps = 0;
  int restarts = 0, reorth_count = 0, deflations = 0;
  bool all_converged = false;
  double wall_seconds = 0.0, device_seconds = 0.0;
  int64_t host_syncs = 0, fused_tails = 0;
  std::vector<double> ritz_history, err_history;
  int64_t history_len = 0;
};
SvdlOutput svdl(DevOp* op, const Options& o);

// subspace_iterate, QR variant, device-resident blocks (subspace_driver.cpp)
struct SubspaceOutput {
  std::vector<double> basis, eigvals, singvals, delta_history, invcond_history;
  int64_t iterations = 0, mvps = 0;
  bool converged = false, rank_deficient = false;
};
SubspaceOutput subspace_qr_device(DevOp* op, int64_t k, double tol, int64_t max_iter,
                                  uint64_t seed, bool scaled_delta);

}  // namespace gkb
