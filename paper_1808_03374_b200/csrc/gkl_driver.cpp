// GKL driver (reference gkl.hpp / gkl.cpp) with device-resident Krylov
// bases: U (reference left basis, SNP side, length m) is sharded by rows like
// the operator, V (sample side, length n, plus the pending vector) is
// replicated on every shard. B, the couplings, the omega rows, Ritz
// extraction and the small SVD stay on the host; every host decision reads
// device scalars (norms) after a fixed-order device reduction, all of which
// are identical on every shard/rank.
//
// Control flow, constants and update order follow gkl.cpp line by line; the
// line references below are to /root/reference/proj/src/gkl.cpp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "host.hpp"

namespace gkb {

namespace {

const double kEps = std::numeric_limits<double>::epsilon();
const double kBreakdownFactor = std::pow(kEps, 2.0 / 3.0);  // gkl.cpp:19
const double kOneSidedGuard = 1.0 / std::sqrt(kEps);        // gkl.cpp:21
const double kCgs2Eta = 0.70710678118654752440;             // orth.hpp:11

double eps_level(int64_t m, int64_t n) {  // gkl.cpp:23-25
  return kEps * std::sqrt(static_cast<double>(std::max(m, n)));
}

bool monitors_side(bool left, int64_t m, int64_t n, const Options& o, double norm_scale) {
  if (!o.one_sided || norm_scale > kOneSidedGuard) return true;  // gkl.cpp:27-33
  return left ? m <= n : n < m;
}

}  // namespace

Options options_from(const gkb_gkl_options* o) {
  Options r;
  if (!o) return r;
  r.k = o->k;
  r.tol = o->tol;
  r.max_mvps = o->max_mvps;
  r.full = o->reorth == 0;
  r.omega = o->omega;
  r.one_sided = o->one_sided != 0;
  r.thick = o->restart == 1;
  r.max_subspace = o->max_subspace;
  r.keep = o->keep;
  r.seed = o->seed;
  r.record_history = o->record_history != 0;
  r.omega_recurrence = o->omega_recurrence;
  return r;
}

// GklOptions::validate (gkl.cpp:53-73), same messages.
void validate_options(const Options& o, int64_t m, int64_t n) {
  const int64_t minmn = std::min(m, n);
  if (m <= 0 || n <= 0) fail(GKB_EINVAL, "svdl: operator has an empty dimension");
  if (o.k < 1 || o.k > minmn) fail(GKB_EINVAL, "svdl: k must lie in [1, min(m, n)]");
  if (!(o.tol > 0.0)) fail(GKB_EINVAL, "svdl: tol must be positive");
  if (o.max_mvps < 2) fail(GKB_EINVAL, "svdl: max_mvps must allow at least one step");
  if (!o.full && !(o.omega > 0.0)) fail(GKB_EINVAL, "svdl: omega must be positive");
  if (o.thick) {
    if (o.keep < o.k) fail(GKB_EINVAL, "svdl: keep must be at least k");
    if (o.keep >= o.max_subspace) fail(GKB_EINVAL, "svdl: keep must be below max_subspace");
    if (o.max_subspace > minmn) fail(GKB_EINVAL, "svdl: max_subspace cannot exceed min(m, n)");
  }
}

// ---------------------------------------------------------------- Lanczos
// LanczosFactorization ctor (gkl.cpp:75-98)
Lanczos::Lanczos(DevOp* op, int64_t capacity, const double* start, uint64_t rng_seed)
    : rng(rng_seed), op_(op), ctx_(op->ctx), m_(op->m), n_(op->n) {
  if (m_ <= 0 || n_ <= 0) fail(GKB_EINVAL, "LanczosFactorization: empty dimensions");
  cap_ = std::min(capacity, std::min(m_, n_));
  if (cap_ < 1) fail(GKB_EINVAL, "LanczosFactorization: capacity < 1");
  double nrm = 0.0;
  for (int64_t i = 0; i < n_; ++i) nrm += start[i] * start[i];
  nrm = std::sqrt(nrm);
  if (!(nrm > 0.0)) fail(GKB_EINVAL, "LanczosFactorization: zero start vector");
  const int L = (int)ctx_->shards.size();
  U_.assign(L, nullptr);
  U2_.assign(L, nullptr);
  V_.assign(L, nullptr);
  V2_.assign(L, nullptr);
  w_.assign(L, nullptr);
  z_.assign(L, nullptr);
  cbuf_.assign(L, nullptr);
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    const size_t r = (size_t)std::max<int64_t>(op_->rows(i), 1);
    // bases and work vectors: stream-ordered from the device pool (an svdl
    // call allocates them; repeated solves reuse the pooled memory)
    cudaStream_t st = ctx_->shards[i].stream;
    auto pool_alloc = [&](double** p, size_t doubles) {
      GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(double) * doubles, st));
    };
    pool_alloc(&U_[i], r * (size_t)cap_);
    pool_alloc(&U2_[i], r * (size_t)cap_);
    pool_alloc(&V_[i], (size_t)n_ * (size_t)(cap_ + 1));
    pool_alloc(&V2_[i], (size_t)n_ * (size_t)(cap_ + 1));
    pool_alloc(&w_[i], r);
    pool_alloc(&z_[i], (size_t)n_);
    pool_alloc(&cbuf_[i], (size_t)(cap_ + 2));
    const int64_t need = dev::red_blocks(std::max<int64_t>(op_->rows(i), n_)) * (cap_ + 4) + 64;
    ctx_->shards[i].ensure_partial(need);
    // result slots: cgs2 against up to cap + 1 columns writes 2 (cap + 1) + 5
    ctx_->shards[i].ensure_res(2 * cap_ + 64);
  }
  B_.assign((size_t)(cap_ * cap_), 0.0);
  coupling_.assign((size_t)cap_, 0.0);
  mu_.assign((size_t)(cap_ + 2), 0.0);
  mu_next_.assign((size_t)(cap_ + 2), 0.0);
  nu_.assign((size_t)(cap_ + 1), 0.0);
  nu_next_.assign((size_t)(cap_ + 1), 0.0);
  ctx_->set_device(0);
  GKB_CUDA(cudaEventCreateWithFlags(&ev_left_, cudaEventDisableTiming));
  GKB_CUDA(cudaEventCreateWithFlags(&ev_right_, cudaEventDisableTiming));
  {
    const char* e = getenv("GKB_NO_SPECULATE");  // sequential order (equivalence tests)
    speculate_ = !(e && e[0] == '1');
  }
  std::vector<double> v0(start, start + n_);
  for (auto& x : v0) x /= nrm;
  host_to_all(v0.data(), n_, V_);
  mu_[0] = 1.0;
  ctx_->sync_all();
}

Lanczos::~Lanczos() {
  for (size_t i = 0; i < U_.size(); ++i) {
    cudaSetDevice(ctx_->shards[i].dev);
    cudaStream_t st = ctx_->shards[i].stream;
    for (double* p : {U_[i], U2_[i], V_[i], V2_[i], w_[i], z_[i], cbuf_[i]})
      if (p) cudaFreeAsync(p, st);  // back to the pool, stream-ordered
    cudaStreamSynchronize(st);
    if (i < tmp_small_.size() && tmp_small_[i]) cudaFree(tmp_small_[i]);
  }
  for (size_t i = 0; i < ctl_d_.size(); ++i)
    if (ctl_d_[i]) {
      cudaSetDevice(ctx_->shards[i].dev);
      cudaFree(ctl_d_[i]);
    }
  if (ctl_up_) cudaFreeHost(ctl_up_);
  if (ctl_down_) cudaFreeHost(ctl_down_);
  for (double* p : ring_slot_)
    if (p) cudaFreeHost(p);
  for (cudaEvent_t e : ring_ev_)
    if (e) cudaEventDestroy(e);
  if (ev_left_) cudaEventDestroy(ev_left_);
  if (ev_right_) cudaEventDestroy(ev_right_);
  if (tlog_) {  // GKB_RTAIL_TLOG: mean SM cycles per phase of the fused right tail
    unsigned long long h[16] = {};
    cudaSetDevice(ctx_->shards[0].dev);
    cudaMemcpy(h, tlog_, sizeof(h), cudaMemcpyDeviceToHost);
    static const char* names[] = {"load", "partials", "barrier", "finalize", "second pass",
                                  "omega", "gt", "gt-bar", "end", "gt-fin", "gn", "gn-bar+fin",
                                  "pass2", "#cgs2", "#pass2"};
    fprintf(stderr, "[gkb] fused right tail, %llu launches, mean cycles per phase:", h[15]);
    for (int k = 0; k < 15; ++k)
      fprintf(stderr, " %s %.0f", names[k],
              k >= 13 ? (double)h[k] : (h[15] ? (double)h[k] / (double)h[15] : 0.0));
    fprintf(stderr, "\n");
    cudaFree(tlog_);
  }
}

// Small host->device uploads (coupling coefficients, restart matrices, start
// vectors) go through a ring of pinned staging slots; a slot is reused only
// after its previous copies (recorded events) have completed, so uploads never
// synchronize the streams.
void Lanczos::host_to_all(const double* h, int64_t count, std::vector<double*>& dst) {
  if (count == 0) return;
  const int L = (int)dst.size();
  if (ring_cap_ < count || (int)ring_ev_.size() != kRing * L) {
    ctx_->sync_all();
    for (double* p : ring_slot_)
      if (p) GKB_CUDA(cudaFreeHost(p));
    for (cudaEvent_t e : ring_ev_)
      if (e) cudaEventDestroy(e);
    ring_cap_ = std::max<int64_t>(std::max(count, ring_cap_), 1 << 12);
    ring_slot_.assign(kRing, nullptr);
    ring_ev_.assign((size_t)(kRing * L), nullptr);
    for (int k = 0; k < kRing; ++k)
      GKB_CUDA(cudaMallocHost(&ring_slot_[k], sizeof(double) * (size_t)ring_cap_));
    for (int k = 0; k < kRing; ++k)
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        GKB_CUDA(cudaEventCreateWithFlags(&ring_ev_[k * L + i], cudaEventDisableTiming));
      }
    ring_used_.assign(kRing, 0);
    ring_next_ = 0;
  }
  const int k = ring_next_;
  ring_next_ = (ring_next_ + 1) % kRing;
  if (ring_used_[k])
    for (int i = 0; i < L; ++i) GKB_CUDA(cudaEventSynchronize(ring_ev_[k * L + i]));
  std::memcpy(ring_slot_[k], h, sizeof(double) * (size_t)count);
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    GKB_CUDA(cudaMemcpyAsync(dst[i], ring_slot_[k], sizeof(double) * (size_t)count,
                             cudaMemcpyHostToDevice, ctx_->shards[i].stream));
    GKB_CUDA(cudaEventRecord(ring_ev_[k * L + i], ctx_->shards[i].stream));
  }
  ring_used_[k] = 1;
}

void Lanczos::upload_small(const std::vector<double>& W, std::vector<double*>& dst) {
  const int64_t need = (int64_t)W.size();
  const int L = (int)ctx_->shards.size();
  if (tmp_small_.size() != (size_t)L) tmp_small_.assign(L, nullptr);
  if (tmp_cap_ < need) {
    ctx_->sync_all();
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      if (tmp_small_[i]) GKB_CUDA(cudaFree(tmp_small_[i]));
      GKB_CUDA(cudaMalloc(&tmp_small_[i], sizeof(double) * (size_t)std::max<int64_t>(need, 1024)));
    }
    tmp_cap_ = std::max<int64_t>(need, 1024);
  }
  host_to_all(W.data(), need, tmp_small_);
  dst = tmp_small_;
}

void Lanczos::read_async(int64_t off, int64_t count, cudaEvent_t ev) {
  Shard& s = ctx_->shards[0];
  ctx_->set_device(0);
  GKB_CUDA(cudaMemcpyAsync(s.hres + off, s.dres + off, sizeof(double) * (size_t)count,
                           cudaMemcpyDeviceToHost, s.stream));
  GKB_CUDA(cudaEventRecord(ev, s.stream));
}

void Lanczos::wait_event(cudaEvent_t ev) {
  GKB_CUDA(cudaEventSynchronize(ev));
  ++host_syncs;
}

void Lanczos::read(int64_t count) {
  Shard& s = ctx_->shards[0];
  ctx_->set_device(0);
  GKB_CUDA(cudaMemcpyAsync(s.hres, s.dres, sizeof(double) * (size_t)count, cudaMemcpyDeviceToHost,
                           s.stream));
  GKB_CUDA(cudaStreamSynchronize(s.stream));
  ++host_syncs;
}

// cgs2 (orth.hpp:19-44) on device vectors. Left side (sharded rows):
// partial dot products are summed across shards before use.
double Lanczos::cgs2(Side side, int64_t ncols, const std::vector<double*>& vec) {
  const int L = (int)ctx_->shards.size();
  const auto& Q = basis(side);
  std::vector<double*> dres(L);
  for (int i = 0; i < L; ++i) dres[i] = ctx_->shards[i].dres;
  auto reduce = [&](int64_t off, int64_t cnt) {
    if (side != kLeft) return;
    std::vector<double*> b(L);
    for (int i = 0; i < L; ++i) b[i] = dres[i] + off;
    ctx_->allreduce(b, cnt);
  };
  if (ncols == 0) {
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      dev::nrm2sq(vec[i], len(side, i), ctx_->shards[i].rs, dres[i], ctx_->shards[i].stream);
    }
    reduce(0, 1);
    read(1);
    return std::sqrt(ctx_->shards[0].hres[0]);
  }
  // pass 1: c = Q^T v and ||v||^2 in one sweep, then v -= Q c with ||v||^2
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    Shard& s = ctx_->shards[i];
    dev::gemv_t(Q[i], ld(side, i), len(side, i), ncols, vec[i], true, s.rs, dres[i], s.stream);
  }
  reduce(0, ncols + 1);
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    Shard& s = ctx_->shards[i];
    dev::gemv_n(Q[i], ld(side, i), len(side, i), ncols, dres[i], vec[i], 1.0, -1.0, true, s.rs,
                dres[i] + ncols + 1, s.stream);
  }
  reduce(ncols + 1, 2);
  read(ncols + 3);
  const double norm_before = std::sqrt(ctx_->shards[0].hres[ncols]);
  double norm_after = std::sqrt(ctx_->shards[0].hres[ncols + 2]);
  if (norm_after < kCgs2Eta * norm_before) {
    const int64_t o = ncols + 3;
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      Shard& s = ctx_->shards[i];
      dev::gemv_t(Q[i], ld(side, i), len(side, i), ncols, vec[i], false, s.rs, dres[i] + o, s.stream);
    }
    reduce(o, ncols);
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      Shard& s = ctx_->shards[i];
      dev::gemv_n(Q[i], ld(side, i), len(side, i), ncols, dres[i] + o, vec[i], 1.0, -1.0, true, s.rs,
                  dres[i] + o + ncols, s.stream);
    }
    reduce(o + ncols, 2);
    read(o + ncols + 2);
    norm_after = std::sqrt(ctx_->shards[0].hres[o + ncols + 1]);
  }
  return norm_after;
}

// Host-side prediction used to decide whether to launch the right half-step
// before alpha is known: the left omega estimate (the same recurrence as
// partial_reorth_update) evaluated with a pessimistic alpha (half the previous
// one). Only a hint -- a wrong guess costs one discarded K2, never a result.
bool Lanczos::left_reorth_unlikely(const Options& o, double norm_scale) const {
  const int64_t j = j_;
  if (j == 0) return false;
  if (!monitors_side(true, m_, n_, o, norm_scale)) return true;
  const double lvl = eps_level(m_, n_);
  const double tau = 2.0 * lvl * norm_scale + lvl;
  const double guess = 0.5 * Bc(j - 1, j - 1);
  const double denom = std::max(guess, tau + kEps);
  for (int64_t i = 0; i < j; ++i) {
    double acc = 0.0;
    for (int64_t c = i; c < j; ++c) acc += std::abs(Bc(i, c)) * mu_[c];
    if (std::min(1.0, (acc + tau) / denom) > o.omega) return false;
  }
  return true;
}

// partial_reorth_update (gkl.cpp:112-176): omega recurrences on the host,
// device cgs2 when the estimate crosses omega.
bool Lanczos::partial_reorth_update(Side side, const std::vector<double*>& cand, double cand_coeff,
                                    const Options& o, double norm_scale, double* new_norm) {
  const int64_t j = j_;
  const double lvl = eps_level(m_, n_);
  const double tau = 2.0 * lvl * norm_scale + lvl;
  const double denom = std::max(cand_coeff, tau + kEps);
  double worst = 0.0;
  if (side == kLeft) {
    for (int64_t i = 0; i < j; ++i) {
      double acc = 0.0;
      for (int64_t c = i; c < j; ++c) acc += std::abs(Bc(i, c)) * mu_[c];
      if (o.omega_recurrence == 1) {
        // alpha u_new = X v - sum_c coupling_c u_c: the u_i component of each
        // subtracted coupling_c u_c (c != i) is bounded by |coupling_c| * nu,
        // nu being the committed level of the newest u (or the restart carry).
        for (int64_t c = 0; c < j; ++c)
          if (c != i && coupling_[c] != 0.0) acc += std::abs(coupling_[c]) * nu_[std::min(c, i)];
      }
      const double est = std::min(1.0, (acc + tau) / denom);
      nu_next_[i] = est;
      worst = std::max(worst, est);
    }
    nu_next_[j] = 1.0;
    if (worst > o.omega && monitors_side(true, m_, n_, o, norm_scale)) {
      // ||w|| after the passes (gkl.cpp:244 recomputes w.norm(); cgs2 returns it)
      *new_norm = cgs2(kLeft, j, cand);
      for (int64_t i = 0; i < j; ++i) nu_next_[i] = lvl;
      return true;
    }
    return false;
  }
  const double alpha_last = Bc(j - 1, j - 1);
  for (int64_t i = 0; i < j; ++i) {
    double acc = 0.0;
    if (i == j - 1) {
      for (int64_t r = 0; r + 1 < j; ++r) acc += std::abs(Bc(r, i)) * nu_[r];
    } else {
      for (int64_t r = 0; r <= i; ++r) acc += std::abs(Bc(r, i)) * nu_[r];
      acc += alpha_last * mu_[i];
    }
    const double est = std::min(1.0, (acc + tau) / denom);
    mu_next_[i] = est;
    worst = std::max(worst, est);
  }
  mu_next_[j] = 1.0;
  if (worst > o.omega && monitors_side(false, m_, n_, o, norm_scale)) {
    *new_norm = cgs2(kRight, j, cand);  // = z.norm() after the passes (gkl.cpp:290)
    for (int64_t i = 0; i < j; ++i) mu_next_[i] = lvl;
    return true;
  }
  return false;
}

// deflate_right (gkl.cpp:178-204)
void Lanczos::deflate_right() {
  ++version_;
  const int64_t j = j_;
  const double lvl = eps_level(m_, n_);
  const int L = (int)ctx_->shards.size();
  std::fill(coupling_.begin(), coupling_.begin() + j, 0.0);
  if (j < n_) {
    std::vector<double> v((size_t)n_);
    for (int attempt = 0; attempt < 4; ++attempt) {
      for (int64_t i = 0; i < n_; ++i) v[i] = rng.uniform_symmetric();
      host_to_all(v.data(), n_, z_);
      const double nrm = cgs2(kRight, j, z_);
      if (nrm > 1e-3 * std::sqrt(static_cast<double>(n_))) {
        for (int i = 0; i < L; ++i) {
          ctx_->set_device(i);
          dev::div_copy(z_[i], nrm, V_[i] + j * n_, n_, ctx_->shards[i].stream);
        }
        std::fill(mu_.begin(), mu_.begin() + j, lvl);
        mu_[j] = 1.0;
        right_exhausted_ = false;
        return;
      }
    }
  }
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    GKB_CUDA(cudaMemsetAsync(V_[i] + j * n_, 0, sizeof(double) * (size_t)n_, ctx_->shards[i].stream));
  }
  std::fill(mu_.begin(), mu_.begin() + j + 1, lvl);
  right_exhausted_ = true;
}

// Right half-step kernels after alpha is fixed: u_s = w / alpha (or
// w / sqrt(dres[nidx]) on the device when `dev_alpha`), z = X^T u_s (cross-
// shard sum inside adjoint_dev), then in partial mode z -= alpha v_s with
// both norms into dres[kRightSlot..+1] and their D2H + ev_right_.
void Lanczos::launch_right(int64_t s, const std::vector<double*>& dres, int64_t nidx,
                           bool dev_alpha, double alpha, bool partial) {
  const int L = (int)ctx_->shards.size();
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    const int64_t r = op_->rows(i);
    if (dev_alpha)
      dev::div_copy_dsq(w_[i], dres[i] + nidx, U_[i] + s * r, r, ctx_->shards[i].stream);
    else
      dev::div_copy(w_[i], alpha, U_[i] + s * r, r, ctx_->shards[i].stream);
  }
  std::vector<const double*> uin(L);
  for (int i = 0; i < L; ++i) uin[i] = U_[i] + s * op_->rows(i);
  op_->adjoint_dev(uin, z_);
  if (!partial) return;
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    Shard& sh = ctx_->shards[i];
    if (dev_alpha)
      dev::axpy_norms_dsq(dres[i] + nidx, V_[i] + s * n_, z_[i], n_, sh.rs, dres[i] + kRightSlot,
                          sh.stream);
    else
      dev::axpy_norms(alpha, V_[i] + s * n_, z_[i], n_, sh.rs, dres[i] + kRightSlot, sh.stream);
  }
  read_async(kRightSlot, 2, ev_right_);
}

// bidiag_step (gkl.cpp:206-312)
StepInfo Lanczos::step(const Options& o, double norm_scale, int64_t* mvp_counter) {
  ++version_;
  const int64_t s = j_;
  if (s >= cap_ || s >= std::min(m_, n_))
    fail(GKB_ELOGIC, "bidiag_step: factorization cannot grow further");
  if (right_exhausted_) fail(GKB_ELOGIC, "bidiag_step: right side exhausted");
  const int L = (int)ctx_->shards.size();
  StepInfo info;
  const double breakdown_tol = kBreakdownFactor * norm_scale;
  const double lvl = eps_level(m_, n_);
  const bool full = o.full;
  std::vector<double*> dres(L);
  for (int i = 0; i < L; ++i) dres[i] = ctx_->shards[i].dres;
  auto reduce_left = [&](int64_t off, int64_t cnt) {
    std::vector<double*> b(L);
    for (int i = 0; i < L; ++i) b[i] = dres[i] + off;
    ctx_->allreduce(b, cnt);
  };
  bool spec = false;  // right half already launched with the device-side alpha

  // Left half-step: alpha u_{s+1} = X v_pending - U coupling.
  {
    std::vector<const double*> vin(L);
    for (int i = 0; i < L; ++i) vin[i] = V_[i] + s * n_;
    op_->apply_dev(vin, w_);
    if (mvp_counter) ++*mvp_counter;
  }
  double alpha;
  if (full) {
    alpha = cgs2(kLeft, s, w_);
  } else {
    int64_t lo = -1, hi = -1;
    for (int64_t i = 0; i < s; ++i)
      if (coupling_[i] != 0.0) {
        if (lo < 0) lo = i;
        hi = i;
      }
    int64_t nidx;  // dres[nidx] = alpha_cand^2 on every shard
    if (lo < 0) {
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        dev::nrm2sq(w_[i], op_->rows(i), ctx_->shards[i].rs, dres[i], ctx_->shards[i].stream);
      }
      reduce_left(0, 1);
      nidx = 0;
    } else {
      std::vector<double> cf(coupling_.begin() + lo, coupling_.begin() + hi + 1);
      host_to_all(cf.data(), hi - lo + 1, cbuf_);
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        Shard& sh = ctx_->shards[i];
        const int64_t r = op_->rows(i);
        dev::gemv_n(U_[i] + lo * r, r, r, hi - lo + 1, cbuf_[i], w_[i], 1.0, -1.0, true, sh.rs,
                    dres[i], sh.stream);
      }
      reduce_left(0, 2);
      nidx = 1;
    }
    // The norms go to the host asynchronously; meanwhile the right half-step
    // is launched with alpha = sqrt(dres[nidx]) taken on the device -- the
    // same IEEE sqrt the host applies below, so every result is bitwise what
    // the sequential order produces. It is discarded (and redone below) when
    // the host's decisions change w: second pass or reorthogonalization.
    read_async(0, nidx + 1, ev_left_);
    if (speculate_ && lo < 0 && left_reorth_unlikely(o, norm_scale)) {
      launch_right(s, dres, nidx, true, 0.0, true);
      spec = true;
    }
    wait_event(ev_left_);
    const double w_norm0 = std::sqrt(ctx_->shards[0].hres[0]);
    double alpha_cand = std::sqrt(ctx_->shards[0].hres[nidx]);
    if (alpha_cand < kCgs2Eta * w_norm0) {
      spec = false;
      // Local (modified) second pass over the structural pattern.
      for (int64_t c = 0; c < s; ++c) {
        if (coupling_[c] == 0.0) continue;
        for (int i = 0; i < L; ++i) {
          ctx_->set_device(i);
          Shard& sh = ctx_->shards[i];
          const int64_t r = op_->rows(i);
          dev::dot(U_[i] + c * r, w_[i], r, sh.rs, dres[i] + 8, sh.stream);
        }
        reduce_left(8, 1);
        for (int i = 0; i < L; ++i) {
          ctx_->set_device(i);
          const int64_t r = op_->rows(i);
          dev::axpy_dev(dres[i] + 8, U_[i] + c * r, w_[i], r, ctx_->shards[i].stream);
        }
      }
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        dev::nrm2sq(w_[i], op_->rows(i), ctx_->shards[i].rs, dres[i], ctx_->shards[i].stream);
      }
      reduce_left(0, 1);
      read(1);
      alpha_cand = std::sqrt(ctx_->shards[0].hres[0]);
    }
    double reorth_norm = 0.0;
    if (partial_reorth_update(kLeft, w_, alpha_cand, o, norm_scale, &reorth_norm)) {
      spec = false;
      info.reorth_left = true;
      alpha_cand = reorth_norm;
    }
    alpha = alpha_cand;
    // (a speculation that turned out wrong is simply overwritten: stream order)
    if (spec) ++spec_hits; else if (speculate_) ++spec_misses;
  }
  if (!(alpha > breakdown_tol)) {
    info.status = 1;
    return info;  // nothing appended (a speculative u_s / z is unused scratch)
  }
  info.alpha = alpha;
  if (!spec) launch_right(s, dres, 0, false, alpha, !full);
  if (mvp_counter) ++*mvp_counter;
  for (int64_t i = 0; i < s; ++i) B(i, s) = coupling_[i];
  B(s, s) = alpha;
  if (full) {
    std::fill(nu_.begin(), nu_.begin() + s, lvl);
    nu_[s] = 1.0;
  } else {
    std::copy(nu_next_.begin(), nu_next_.begin() + s + 1, nu_.begin());
  }
  j_ = s + 1;

  // Right half-step: beta v_new = X^T u_{s+1} - alpha v_pending (z = X^T u
  // and z -= alpha v_s with its norms were launched by launch_right).
  double beta;
  if (full) {
    beta = cgs2(kRight, s + 1, z_);
  } else {
    wait_event(ev_right_);
    const double z_norm0 = std::sqrt(ctx_->shards[0].hres[kRightSlot]);
    double beta_cand = std::sqrt(ctx_->shards[0].hres[kRightSlot + 1]);
    if (beta_cand < kCgs2Eta * z_norm0) {
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        Shard& sh = ctx_->shards[i];
        dev::dot(V_[i] + s * n_, z_[i], n_, sh.rs, dres[i] + 8, sh.stream);
        dev::axpy_dev(dres[i] + 8, V_[i] + s * n_, z_[i], n_, sh.stream);
        dev::nrm2sq(z_[i], n_, sh.rs, dres[i], sh.stream);
      }
      read(1);
      beta_cand = std::sqrt(ctx_->shards[0].hres[0]);
    }
    double reorth_norm = 0.0;
    if (partial_reorth_update(kRight, z_, beta_cand, o, norm_scale, &reorth_norm)) {
      info.reorth_right = true;
      beta_cand = reorth_norm;
    }
    beta = beta_cand;
  }
  std::fill(coupling_.begin(), coupling_.begin() + s + 1, 0.0);
  if (!(beta > breakdown_tol)) {
    info.status = 2;
    deflate_right();
    return info;
  }
  info.beta = beta;
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    dev::div_copy(z_[i], beta, V_[i] + (s + 1) * n_, n_, ctx_->shards[i].stream);
  }
  coupling_[s] = beta;
  if (full) {
    std::fill(mu_.begin(), mu_.begin() + s + 1, lvl);
    mu_[s + 1] = 1.0;
  } else {
    std::copy(mu_next_.begin(), mu_next_.begin() + s + 2, mu_.begin());
  }
  return info;
}

// ---------------------------------------------------------------- device-controlled steps
// The same step as Lanczos::step (gkl.cpp:206-312), enqueued without reading
// anything back: each decision is a ctl kernel (ctl_kernels.cu) writing gates,
// and the kernels of both branches are enqueued with the gate that enables
// them. Kernels and result slots are the host path's, so the values are too.
// The light decisions (L_A, R_A, CG_MID) run inside the reduction that
// produces their inputs (kernels.hpp ctl::Post) unless GKB_NO_CTL_FUSE is set;
// on the left that needs the allreduce in between to be a no-op.
bool Lanczos::fuse_ctl() {
  static const bool on = getenv("GKB_NO_CTL_FUSE") == nullptr;
  return on;
}
bool Lanczos::reduce_local() const {
  return ctx_->spmd_mode ? ctx_->nshards_total == 1 : ctx_->shards.size() == 1;
}

dev::ctl::Params Lanczos::ctl_params(const Options& o, int op, int64_t s) const {
  dev::ctl::Params p{};
  p.op = op;
  p.full = o.full ? 1 : 0;
  p.omega_rec = o.omega_recurrence;
  p.one_sided = o.one_sided ? 1 : 0;
  p.s = s;
  p.m = m_;
  p.n = n_;
  p.cap = cap_;
  p.omega = o.omega;
  p.lvl = eps_level(m_, n_);
  p.bfac = kBreakdownFactor;
  p.guard = kOneSidedGuard;
  p.eta = kCgs2Eta;
  p.eps = kEps;
  p.lo = p.hi = -1;
  p.then_op = -1;
  return p;
}

// cgs2 (orth.hpp:19-44) with its second-pass test on the device; pass 1 runs
// when the int at gate_slot is set (full mode: alive; partial: reorthogonalize).
void Lanczos::cgs2_dev(Side side, int64_t ncols, const std::vector<double*>& vec, int gate_slot,
                       const Options& o, int64_t s, int then_op) {
  using namespace dev::ctl;
  const int L = (int)ctx_->shards.size();
  const auto& Q = basis(side);
  auto res = [&](int i, int64_t off) { return cd(i) + ctl_L_.res + off; };
  auto reduce = [&](int64_t off, int64_t cnt) {
    if (side != kLeft) return;
    std::vector<double*> b(L);
    for (int i = 0; i < L; ++i) b[i] = res(i, off);
    ctx_->allreduce(b, cnt);
  };
  auto ctl = [&](const Params& p) {
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      launch(cd(i), ci(i), p, ctx_->shards[i].stream);
    }
  };
  const int64_t o2 = R_CG + ncols + 3;
  for (int pass = 0; pass < 2; ++pass) {
    const int64_t oc = pass == 0 ? R_CG : o2;  // coefficients (+ ||v||^2 in pass 1)
    const int64_t on = pass == 0 ? R_CG + ncols + 1 : o2 + ncols;  // norms of gemv_n
    const int slot = pass == 0 ? gate_slot : (int)I_GRE2;
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      Shard& sh = ctx_->shards[i];
      dev::gemv_t(Q[i], ld(side, i), len(side, i), ncols, vec[i], pass == 0, sh.rs, res(i, oc),
                  sh.stream, ci(i) + slot);
    }
    reduce(oc, ncols + (pass == 0 ? 1 : 0));
    Params p = ctl_params(o, pass == 0 ? OP_CG_MID : OP_CG_END, s);
    p.ncols = ncols;
    p.side = side == kLeft ? 0 : 1;
    if (pass == 1) p.then_op = then_op;  // e.g. the half-step finalize, same launch
    // pass 1's decision runs in gemv_n's last CTA when no allreduce follows it
    const bool fuse = pass == 0 && fuse_ctl() && (side != kLeft || reduce_local());
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      Shard& sh = ctx_->shards[i];
      Post post;
      post.d = cd(i);
      post.iv = ci(i);
      post.p = p;
      dev::gemv_n(Q[i], ld(side, i), len(side, i), ncols, res(i, oc), vec[i], 1.0, -1.0, true,
                  sh.rs, res(i, on), sh.stream, ci(i) + slot, fuse ? &post : nullptr);
    }
    reduce(on, 2);
    if (!fuse) ctl(p);
  }
}

// The right half-step's tail fused into one launch per shard (the right
// side is replicated: no collective inside it). All shards or none.
bool Lanczos::right_tail_dev(const Options& o, int64_t s) {
  const int L = (int)ctx_->shards.size();
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    Shard& sh = ctx_->shards[i];
    dev::ctl::TailArgs a{cd(i), ci(i), ctl_params(o, dev::ctl::OP_R_B, s), V_[i], z_[i], n_};
    if (i == 0 && getenv("GKB_RTAIL_TLOG")) {  // debug: per-phase cycles of the fused tail
      if (!tlog_) {
        GKB_CUDA(cudaMalloc(&tlog_, 16 * sizeof(unsigned long long)));
        GKB_CUDA(cudaMemset(tlog_, 0, 16 * sizeof(unsigned long long)));
      }
      a.tlog = tlog_;
    }
    if (!dev::ctl::right_tail(a, sh.stream)) {
      if (i == 0) return false;
      fail(GKB_ELOGIC, "fused right tail launched on some shards only");
    }
  }
  ++fused_tails;
  return true;
}

void Lanczos::enqueue_step_dev(const Options& o, int64_t s, int64_t lo, int64_t hi, bool last) {
  using namespace dev::ctl;
  const int L = (int)ctx_->shards.size();
  auto res = [&](int i, int64_t off) { return cd(i) + ctl_L_.res + off; };
  auto reduce_left = [&](int64_t off, int64_t cnt) {
    std::vector<double*> b(L);
    for (int i = 0; i < L; ++i) b[i] = res(i, off);
    ctx_->allreduce(b, cnt);
  };
  auto ctl = [&](const Params& p) {
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      launch(cd(i), ci(i), p, ctx_->shards[i].stream);
    }
  };
  auto scal = [&](int slot) {
    std::vector<const double*> d(L);
    for (int i = 0; i < L; ++i) d[i] = cd(i) + ctl_L_.sc + slot;
    return d;
  };
  auto alive_gates = [&]() {
    std::vector<const int*> g(L);
    for (int i = 0; i < L; ++i) g[i] = ci(i) + I_ALIVE;
    return g;
  };
  // Left half-step: alpha u_{s+1} = X v_s - U coupling.
  {
    std::vector<double*> vcol(L);
    for (int i = 0; i < L; ++i) vcol[i] = V_[i] + s * n_;
    if (v_pending_) {  // v_s = z / beta of the previous step, divided while digitized
      std::vector<const double*> zr(z_.begin(), z_.end());
      op_->apply_dev_div(zr, scal(S_BETA), alive_gates(), vcol, w_);
      v_pending_ = false;
    } else {
      op_->apply_dev(std::vector<const double*>(vcol.begin(), vcol.end()), w_);
    }
  }
  if (o.full) {
    if (s == 0) {
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        Shard& sh = ctx_->shards[i];
        dev::nrm2sq(w_[i], op_->rows(i), sh.rs, res(i, R_N), sh.stream, ci(i) + I_ALIVE);
      }
      reduce_left(R_N, 1);
      Params q = ctl_params(o, OP_SQRT_L, s);
      q.then_op = OP_L_END;
      ctl(q);
    } else {
      cgs2_dev(kLeft, s, w_, I_ALIVE, o, s, OP_L_END);
    }
  } else {
    const bool pat = lo >= 0;
    Params pa = ctl_params(o, OP_L_A, s);
    pa.nidx = pat ? 1 : 0;
    pa.has_pattern = pat ? 1 : 0;
    pa.lo = lo;
    pa.hi = hi;
    const bool fuse = fuse_ctl() && reduce_local();  // decision in the reduction's last CTA
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      Shard& sh = ctx_->shards[i];
      const int64_t r = op_->rows(i);
      Post post;
      post.d = cd(i);
      post.iv = ci(i);
      post.p = pa;
      const Post* pp = fuse ? &post : nullptr;
      if (pat)
        dev::gemv_n(U_[i] + lo * r, r, r, hi - lo + 1, cd(i) + ctl_L_.coup + lo, w_[i], 1.0, -1.0,
                    true, sh.rs, res(i, R_N), sh.stream, ci(i) + I_ALIVE, pp);
      else
        dev::nrm2sq(w_[i], r, sh.rs, res(i, R_N), sh.stream, ci(i) + I_ALIVE, pp);
    }
    reduce_left(R_N, pat ? 2 : 1);
    if (!fuse) ctl(pa);
    if (pat && fuse_ctl()) {  // local second pass over the structural pattern (gkl.cpp:233-242)
      // column c's axpy fused with column c+1's dot (or the final norm): the
      // dot slots alternate so no CTA reads a slot the same launch writes
      auto dslot = [&](int i, int64_t c) { return res(i, R_DOT + (c & 1)); };
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        Shard& sh = ctx_->shards[i];
        const int64_t r = op_->rows(i);
        dev::dot(U_[i] + lo * r, w_[i], r, sh.rs, dslot(i, lo), sh.stream, ci(i) + I_G2PC + lo);
      }
      reduce_left(R_DOT + (lo & 1), 1);
      for (int64_t c = lo; c <= hi; ++c) {
        const bool last = c == hi;
        for (int i = 0; i < L; ++i) {
          ctx_->set_device(i);
          Shard& sh = ctx_->shards[i];
          const int64_t r = op_->rows(i);
          dev::axpy_dot(dslot(i, c), U_[i] + c * r, ci(i) + I_G2PC + c,
                        last ? nullptr : U_[i] + (c + 1) * r, ci(i) + (last ? I_G2P : I_G2PC + c + 1),
                        w_[i], r, sh.rs, last ? res(i, R_N) : dslot(i, c + 1), sh.stream);
        }
        reduce_left(last ? R_N : R_DOT + ((c + 1) & 1), 1);
      }
    } else if (pat) {
      for (int64_t c = lo; c <= hi; ++c) {
        for (int i = 0; i < L; ++i) {
          ctx_->set_device(i);
          Shard& sh = ctx_->shards[i];
          const int64_t r = op_->rows(i);
          dev::dot(U_[i] + c * r, w_[i], r, sh.rs, res(i, R_DOT), sh.stream, ci(i) + I_G2PC + c);
        }
        reduce_left(R_DOT, 1);
        for (int i = 0; i < L; ++i) {
          ctx_->set_device(i);
          const int64_t r = op_->rows(i);
          dev::axpy_dev(res(i, R_DOT), U_[i] + c * r, w_[i], r, ctx_->shards[i].stream,
                        ci(i) + I_G2PC + c);
        }
      }
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        Shard& sh = ctx_->shards[i];
        dev::nrm2sq(w_[i], op_->rows(i), sh.rs, res(i, R_N), sh.stream, ci(i) + I_G2P);
      }
      reduce_left(R_N, 1);
    }
    if (s > 0) {
      ctl(ctl_params(o, OP_L_B, s));
      cgs2_dev(kLeft, s, w_, I_GRE, o, s, OP_L_END);
    } else {  // no basis yet: the omega test has no rows
      Params q = ctl_params(o, OP_L_B, s);
      q.then_op = OP_L_END;
      ctl(q);
    }
  }

  // Right half-step: beta v_{s+1} = X^T u_{s+1} - alpha v_s, u_{s+1} = w / alpha
  // (divided while the adjoint digitizes it unless GKB_NO_CTL_FUSE).
  {
    std::vector<double*> ucol(L);
    for (int i = 0; i < L; ++i) ucol[i] = U_[i] + s * op_->rows(i);
    std::vector<const double*> wr(w_.begin(), w_.end());
    if (fuse_ctl()) {
      op_->adjoint_dev_div(wr, scal(S_ALPHA), alive_gates(), ucol, z_);
    } else {
      for (int i = 0; i < L; ++i) {
        ctx_->set_device(i);
        dev::div_copy_dv(w_[i], cd(i) + ctl_L_.sc + S_ALPHA, ucol[i], op_->rows(i),
                         ctx_->shards[i].stream, ci(i) + I_ALIVE);
      }
      op_->adjoint_dev(std::vector<const double*>(ucol.begin(), ucol.end()), z_);
    }
  }
  if (fuse_ctl() && right_tail_dev(o, s)) {
    // the whole sequence below in one cluster launch (ctl_kernels.cu k_right_tail)
  } else if (!o.full) {
    const bool fuse = fuse_ctl();  // right side: no allreduce before the decision
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      Shard& sh = ctx_->shards[i];
      Post post;
      post.d = cd(i);
      post.iv = ci(i);
      post.p = ctl_params(o, OP_R_A, s);
      dev::axpy_norms_dv(cd(i) + ctl_L_.sc + S_ALPHA, V_[i] + s * n_, z_[i], n_, sh.rs,
                         res(i, R_N), sh.stream, ci(i) + I_ALIVE, fuse ? &post : nullptr);
    }
    if (!fuse) ctl(ctl_params(o, OP_R_A, s));
    for (int i = 0; i < L; ++i) {  // local second pass against v_s (gkl.cpp:277-284)
      ctx_->set_device(i);
      Shard& sh = ctx_->shards[i];
      const int* g = ci(i) + I_G2P;
      dev::dot(V_[i] + s * n_, z_[i], n_, sh.rs, res(i, R_DOT), sh.stream, g);
      if (fuse) {
        dev::axpy_dot(res(i, R_DOT), V_[i] + s * n_, g, nullptr, g, z_[i], n_, sh.rs, res(i, R_N),
                      sh.stream);
      } else {
        dev::axpy_dev(res(i, R_DOT), V_[i] + s * n_, z_[i], n_, sh.stream, g);
        dev::nrm2sq(z_[i], n_, sh.rs, res(i, R_N), sh.stream, g);
      }
    }
    ctl(ctl_params(o, OP_R_B, s));
    cgs2_dev(kRight, s + 1, z_, I_GRE, o, s, OP_R_END);
  } else {
    cgs2_dev(kRight, s + 1, z_, I_ALIVE, o, s, OP_R_END);
  }
  if (fuse_ctl() && !last) {  // v_{s+1} = z / beta: divided by the next step's apply
    v_pending_ = true;
    return;
  }
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    dev::div_copy_dv(z_[i], cd(i) + ctl_L_.sc + S_BETA, V_[i] + (s + 1) * n_, n_,
                     ctx_->shards[i].stream, ci(i) + I_ALIVE);
  }
}

Lanczos::DevRun Lanczos::run_dev(const Options& o, int64_t nsteps, double* norm_scale) {
  const auto t_run0 = std::chrono::steady_clock::now();
  ++version_;
  using namespace dev::ctl;
  const int L = (int)ctx_->shards.size();
  if (ctl_d_.empty()) {
    ctl_L_ = layout(cap_);
    ctl_d_.assign(L, nullptr);
    for (int i = 0; i < L; ++i) {
      ctx_->set_device(i);
      GKB_CUDA(cudaMalloc(&ctl_d_[i], ctl_L_.bytes));
    }
    GKB_CUDA(cudaMallocHost(&ctl_up_, ctl_L_.bytes));
    GKB_CUDA(cudaMallocHost(&ctl_down_, ctl_L_.bytes));
  }
  // host state -> every replica
  double* hd = reinterpret_cast<double*>(ctl_up_);
  int* hi = reinterpret_cast<int*>(hd + ctl_L_.nd);
  std::memset(ctl_up_, 0, ctl_L_.bytes);
  std::copy(B_.begin(), B_.end(), hd + ctl_L_.B);
  std::copy(coupling_.begin(), coupling_.end(), hd + ctl_L_.coup);
  std::copy(mu_.begin(), mu_.end(), hd + ctl_L_.mu);
  std::copy(nu_.begin(), nu_.end(), hd + ctl_L_.nu);
  hd[ctl_L_.sc + S_NS] = *norm_scale;
  hi[I_ALIVE] = 1;
  hi[I_J] = (int)j_;
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    GKB_CUDA(cudaMemcpyAsync(ctl_d_[i], ctl_up_, ctl_L_.bytes, cudaMemcpyHostToDevice,
                             ctx_->shards[i].stream));
  }
  // first step: the coupling pattern of the host state; later steps: {s - 1}
  int64_t lo = -1, hi_c = -1;
  for (int64_t i = 0; i < j_; ++i)
    if (coupling_[i] != 0.0) {
      if (lo < 0) lo = i;
      hi_c = i;
    }
  v_pending_ = false;
  for (int64_t t = 0; t < nsteps; ++t) {
    const int64_t s = j_ + t;
    if (t > 0) lo = hi_c = s - 1;
    enqueue_step_dev(o, s, lo, hi_c, t + 1 == nsteps);
  }
  ctx_->set_device(0);
  Shard& s0 = ctx_->shards[0];
  GKB_CUDA(cudaMemcpyAsync(ctl_down_, ctl_d_[0], ctl_L_.bytes, cudaMemcpyDeviceToHost, s0.stream));
  const auto t_enq = std::chrono::steady_clock::now();
  ctx_->sync_all();
  const auto t_done = std::chrono::steady_clock::now();
  t_enqueue += std::chrono::duration<double>(t_enq - t_run0).count();
  t_wait += std::chrono::duration<double>(t_done - t_enq).count();
  ++host_syncs;
  const double* dd = reinterpret_cast<const double*>(ctl_down_);
  const int* di = reinterpret_cast<const int*>(dd + ctl_L_.nd);
  std::copy(dd + ctl_L_.B, dd + ctl_L_.B + cap_ * cap_, B_.begin());
  std::copy(dd + ctl_L_.coup, dd + ctl_L_.coup + cap_, coupling_.begin());
  std::copy(dd + ctl_L_.mu, dd + ctl_L_.mu + cap_ + 2, mu_.begin());
  std::copy(dd + ctl_L_.nu, dd + ctl_L_.nu + cap_ + 1, nu_.begin());
  *norm_scale = dd[ctl_L_.sc + S_NS];
  j_ = di[I_J];
  DevRun r;
  r.completed = di[I_STEPS];
  r.status = di[I_STATUS];
  r.reorth = di[I_REORTH];
  return r;
}

// ritz_extract (gkl.cpp:314-339)
Ritz Lanczos::ritz_extract(double tol) const {
  Ritz out;
  const int64_t j = j_;
  out.j = j;
  if (j == 0) return out;
  std::vector<double> Bj((size_t)(j * j));
  for (int64_t c = 0; c < j; ++c)
    for (int64_t r = 0; r < j; ++r) Bj[r + c * j] = Bc(r, c);
  out.values.assign((size_t)j, 0.0);
  out.WL.assign((size_t)(j * j), 0.0);
  out.WR.assign((size_t)(j * j), 0.0);
  svd_small(Bj.data(), j, j, out.WL.data(), out.values.data(), out.WR.data());
  out.err_crude.assign((size_t)j, 0.0);
  for (int64_t i = 0; i < j; ++i) {
    double acc = 0.0;
    for (int64_t r = 0; r < j; ++r) acc += out.WL[r + i * j] * coupling_[r];
    out.err_crude[i] = std::abs(acc);
  }
  out.err = out.err_crude;
  for (int64_t i = 0; i < j; ++i) {
    double gap = std::numeric_limits<double>::infinity();
    for (int64_t l = 0; l < j; ++l)
      if (l != i) gap = std::min(gap, std::abs(out.values[l] - out.values[i]));
    if (j > 1 && gap > 10.0 * out.err_crude[i] && gap > 0.0) {
      const double refined = out.err_crude[i] * out.err_crude[i] / gap;
      out.err[i] = std::min(out.err_crude[i], refined);
    }
  }
  const double theta_max = out.values[0];
  out.converged.assign((size_t)j, 0);
  for (int64_t i = 0; i < j; ++i) out.converged[i] = out.err[i] <= tol * theta_max;
  return out;
}

// thick_restart (gkl.cpp:341-378)
void Lanczos::thick_restart(int64_t keep, const Ritz* current) {
  ++version_;
  const int64_t j = j_;
  if (keep < 1 || keep >= j) fail(GKB_EINVAL, "thick_restart: need 1 <= keep < steps");
  const int L = (int)ctx_->shards.size();
  // (the convergence tolerance only sets Ritz::converged: any extract of this
  // factorization has the values and vectors used here)
  Ritz own;
  if (!current || current->j != j) own = ritz_extract(0.0);
  const Ritz& ritz = (current && current->j == j) ? *current : own;
  std::vector<double> rho((size_t)keep);
  for (int64_t i = 0; i < keep; ++i) {
    double acc = 0.0;
    for (int64_t r = 0; r < j; ++r) acc += ritz.WL[r + i * j] * coupling_[r];
    rho[i] = acc;
  }
  // W = [W_L[:, :keep] | W_R[:, :keep]] uploaded once
  std::vector<double> Wup((size_t)(2 * j * keep));
  std::copy(ritz.WL.begin(), ritz.WL.begin() + j * keep, Wup.begin());
  std::copy(ritz.WR.begin(), ritz.WR.begin() + j * keep, Wup.begin() + j * keep);
  std::vector<double*> Wd;
  upload_small(Wup, Wd);
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    cudaStream_t st = ctx_->shards[i].stream;
    const int64_t r = op_->rows(i);
    dev::gemm_small(U_[i], r, r, j, Wd[i], j, keep, U2_[i], r, st);
    dev::gemm_small(V_[i], n_, n_, j, Wd[i] + j * keep, j, keep, V2_[i], n_, st);
    GKB_CUDA(cudaMemcpyAsync(V2_[i] + keep * n_, V_[i] + j * n_, sizeof(double) * (size_t)n_,
                             cudaMemcpyDeviceToDevice, st));
    std::swap(U_[i], U2_[i]);
    std::swap(V_[i], V2_[i]);
  }
  std::fill(B_.begin(), B_.end(), 0.0);
  for (int64_t i = 0; i < keep; ++i) B(i, i) = ritz.values[i];
  std::fill(coupling_.begin(), coupling_.end(), 0.0);
  for (int64_t i = 0; i < keep; ++i) coupling_[i] = rho[i];
  j_ = keep;
  const double lvl = eps_level(m_, n_);
  const double scale = std::sqrt(static_cast<double>(j));
  const double mmax = *std::max_element(mu_.begin(), mu_.begin() + j);
  const double nmax = *std::max_element(nu_.begin(), nu_.begin() + j);
  const double mu_carry = std::min(1.0, scale * mmax + lvl);
  const double nu_carry = std::min(1.0, scale * nmax + lvl);
  std::fill(mu_.begin(), mu_.begin() + keep, mu_carry);
  mu_[keep] = 1.0;
  std::fill(nu_.begin(), nu_.begin() + keep, nu_carry);
}

// compress_exhausted (gkl.cpp:380-409)
void Lanczos::compress_exhausted() {
  ++version_;
  const int64_t j = j_;
  if (j == 0) return;
  const int L = (int)ctx_->shards.size();
  std::vector<double> aug((size_t)(j * (j + 1)));
  for (int64_t c = 0; c < j; ++c)
    for (int64_t r = 0; r < j; ++r) aug[r + c * j] = Bc(r, c);
  for (int64_t r = 0; r < j; ++r) aug[r + j * j] = coupling_[r];
  std::vector<double> SU((size_t)(j * j)), Ss((size_t)j), SV((size_t)((j + 1) * j));
  svd_small(aug.data(), j, j + 1, SU.data(), Ss.data(), SV.data());
  std::vector<double> Wup(SU);
  Wup.insert(Wup.end(), SV.begin(), SV.end());
  std::vector<double*> Wd;
  upload_small(Wup, Wd);
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    cudaStream_t st = ctx_->shards[i].stream;
    const int64_t r = op_->rows(i);
    dev::gemm_small(U_[i], r, r, j, Wd[i], j, j, U2_[i], r, st);
    dev::gemm_small(V_[i], n_, n_, j + 1, Wd[i] + j * j, j + 1, j, V2_[i], n_, st);
    GKB_CUDA(cudaMemsetAsync(V2_[i] + j * n_, 0, sizeof(double) * (size_t)n_, st));
    std::swap(U_[i], U2_[i]);
    std::swap(V_[i], V2_[i]);
  }
  std::fill(B_.begin(), B_.end(), 0.0);
  for (int64_t i = 0; i < j; ++i) B(i, i) = Ss[i];
  std::fill(coupling_.begin(), coupling_.end(), 0.0);
  right_exhausted_ = true;
  const double lvl = eps_level(m_, n_);
  std::fill(mu_.begin(), mu_.begin() + j + 1, lvl);
  std::fill(nu_.begin(), nu_.begin() + j, lvl);
}

// Gathers a left-side (sharded rows) block of `ncols` columns, ld = rows(i),
// into host column-major m x ncols.
static void gather_left(Context* ctx, DevOp* op, const std::vector<double*>& src, int64_t ncols,
                        double* host) {
  const int L = (int)ctx->shards.size();
  const int64_t m = op->m;
  if (ncols == 0) return;
  if (ctx->spmd_mode && ctx->nshards_total > 1) {
    ctx->set_device(0);
    Shard& s = ctx->shards[0];
    DevScratch fhold;  // RAII: freed if the allreduce or a copy throws
    GKB_CUDA(cudaMalloc(&fhold.p, sizeof(double) * (size_t)(m * ncols)));
    double* full = fhold.as<double>();
    GKB_CUDA(cudaMemsetAsync(full, 0, sizeof(double) * (size_t)(m * ncols), s.stream));
    const int64_t r = op->rows(0);
    if (r > 0)
      GKB_CUDA(cudaMemcpy2DAsync(full + op->row0(0), sizeof(double) * (size_t)m, src[0],
                                 sizeof(double) * (size_t)r, sizeof(double) * (size_t)r,
                                 (size_t)ncols, cudaMemcpyDeviceToDevice, s.stream));
    ctx->allreduce({full}, m * ncols);
    GKB_CUDA(cudaMemcpyAsync(host, full, sizeof(double) * (size_t)(m * ncols),
                             cudaMemcpyDeviceToHost, s.stream));
    GKB_CUDA(cudaStreamSynchronize(s.stream));
    return;
  }
  if (L == 1) {  // rows(0) == m: one contiguous block
    ctx->set_device(0);
    ctx->sync_all();
    d2h_staged(ctx->shards[0], host, src[0], sizeof(double) * (size_t)(m * ncols));
    return;
  }
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    const int64_t r = op->rows(i);
    if (r == 0) continue;
    GKB_CUDA(cudaMemcpy2DAsync(host + op->row0(i), sizeof(double) * (size_t)m, src[i],
                               sizeof(double) * (size_t)r, sizeof(double) * (size_t)r,
                               (size_t)ncols, cudaMemcpyDeviceToHost, ctx->shards[i].stream));
  }
  ctx->sync_all();
}

void Lanczos::get(double* U, double* V, double* B, double* coupling, double* om_left,
                  double* om_right) {
  ctx_->sync_all();
  const int64_t j = j_;
  if (U) gather_left(ctx_, op_, U_, j, U);
  if (V) {
    ctx_->set_device(0);
    GKB_CUDA(cudaMemcpyAsync(V, V_[0], sizeof(double) * (size_t)(n_ * (j + 1)),
                             cudaMemcpyDeviceToHost, ctx_->shards[0].stream));
    GKB_CUDA(cudaStreamSynchronize(ctx_->shards[0].stream));
  }
  if (B)
    for (int64_t c = 0; c < j; ++c)
      for (int64_t r = 0; r < j; ++r) B[r + c * j] = Bc(r, c);
  if (coupling) std::copy(coupling_.begin(), coupling_.begin() + j, coupling);
  if (om_left) std::copy(nu_.begin(), nu_.begin() + j, om_left);
  if (om_right) std::copy(mu_.begin(), mu_.begin() + j + 1, om_right);
}

void Lanczos::ritz_vectors(const Ritz& r, int64_t kc, double* outU, double* outV) {
  const int64_t j = j_;
  if (kc == 0 || j == 0) return;
  const int L = (int)ctx_->shards.size();
  std::vector<double> Wup((size_t)(2 * j * kc));
  std::copy(r.WL.begin(), r.WL.begin() + j * kc, Wup.begin());
  std::copy(r.WR.begin(), r.WR.begin() + j * kc, Wup.begin() + j * kc);
  std::vector<double*> Wd;
  upload_small(Wup, Wd);
  for (int i = 0; i < L; ++i) {
    ctx_->set_device(i);
    cudaStream_t st = ctx_->shards[i].stream;
    const int64_t rr = op_->rows(i);
    dev::gemm_small(U_[i], rr, rr, j, Wd[i], j, kc, U2_[i], rr, st);
    dev::gemm_small(V_[i], n_, n_, j, Wd[i] + j * kc, j, kc, V2_[i], n_, st);
  }
  ctx_->sync_all();
  if (outU) gather_left(ctx_, op_, U2_, kc, outU);
  if (outV) {
    ctx_->set_device(0);
    d2h_staged(ctx_->shards[0], outV, V2_[0], sizeof(double) * (size_t)(n_ * kc));
  }
}

// ---------------------------------------------------------------- svdl
// svdl (gkl.cpp:416-514)
SvdlOutput svdl(DevOp* op, const Options& o) {
  const auto t_start = std::chrono::steady_clock::now();
  const int64_t m = op->m, n = op->n;
  validate_options(o, m, n);
  const int64_t minmn = std::min(m, n);
  const int64_t cap = o.thick ? o.max_subspace : minmn;

  int64_t mvps = 0;
  Rng start_rng(o.seed);
  std::vector<double> v0((size_t)n);
  for (int64_t i = 0; i < n; ++i) v0[i] = start_rng.uniform_symmetric();
  // The deflation draws continue the same stream (gkl.cpp:427-430, :189).
  Lanczos f(op, cap, v0.data(), 0);
  f.rng = start_rng;

  Context* ctx = op->ctx;
  cudaEvent_t e0, e1;
  ctx->set_device(0);
  GKB_CUDA(cudaEventCreate(&e0));
  GKB_CUDA(cudaEventCreate(&e1));
  GKB_CUDA(cudaEventRecord(e0, ctx->shards[0].stream));

  SvdlOutput out;
  double t_extract = 0.0, t_restart = 0.0;  // host phases (GKB_VERBOSE)
  double norm_scale = 0.0;
  Ritz ritz;
  int consecutive_breakdowns = 0;
  int64_t ritz_version = -1;  // factorization version the current `ritz` was extracted from
  auto extract = [&]() {
    if (ritz_version == f.version()) {  // unchanged since the last extraction: replay it
      if (o.record_history) {
        const size_t h = out.ritz_history.size();
        for (int64_t i = 0; i < o.k; ++i) {
          out.ritz_history.push_back(out.ritz_history[h - (size_t)o.k + (size_t)i]);
          out.err_history.push_back(out.err_history[h - (size_t)o.k + (size_t)i]);
        }
        ++out.history_len;
      }
      return;
    }
    ritz_version = f.version();
    ritz = f.ritz_extract(o.tol);
    if (!ritz.values.empty()) norm_scale = std::max(norm_scale, ritz.values[0]);
    if (o.record_history) {
      for (int64_t i = 0; i < o.k; ++i) {
        out.ritz_history.push_back(i < ritz.j ? ritz.values[i] : std::nan(""));
        out.err_history.push_back(i < ritz.j ? ritz.err[i] : std::nan(""));
      }
      ++out.history_len;
    }
  };
  auto top_k_converged = [&]() {
    if (f.steps() < o.k || ritz.j < o.k) return false;
    for (int64_t i = 0; i < o.k; ++i)
      if (!ritz.converged[i]) return false;
    return true;
  };

  // Device-controlled steps (one read-back per restart cycle) unless
  // GKB_HOST_STEP=1; without restarts the convergence test reads B after every
  // step, so that mode uses them only while the factorization is small.
  bool dev_steps = o.thick || cap <= 128;
  if (const char* e = getenv("GKB_HOST_STEP"))
    if (e[0] == '1') dev_steps = false;
  while (true) {
    if (f.steps() >= minmn) break;  // factorization complete
    if (mvps + 2 > o.max_mvps) break;
    if (f.right_exhausted()) break;
    if (dev_steps) {
      // steps until the next host decision: the restart point (thick) or the
      // per-step convergence test; never past the mvp budget
      int64_t nmax = o.thick ? o.max_subspace - f.steps() : 1;
      nmax = std::min(nmax, minmn - f.steps());
      nmax = std::min(nmax, (o.max_mvps - mvps) / 2);
      nmax = std::max<int64_t>(nmax, 1);
      const Lanczos::DevRun r = f.run_dev(o, nmax, &norm_scale);
      mvps += 2 * r.completed + (r.status == 1 ? 1 : 0);
      out.steps += r.completed;
      out.reorth_count += (int)r.reorth;
      if (r.completed > (r.status == 2 ? 1 : 0)) consecutive_breakdowns = 0;
      if (r.status == 1) {  // as below: alpha breakdown
        ++out.deflations;
        ++consecutive_breakdowns;
        f.compress_exhausted();
        extract();
        if (top_k_converged() || consecutive_breakdowns > 3) break;
        f.deflate_right();
        continue;
      }
      if (r.status == 2) {  // beta breakdown: step() deflates before returning
        ++out.deflations;
        ++consecutive_breakdowns;
        f.deflate_right();
      }
      if (!o.thick) {
        extract();
        if (top_k_converged()) break;
      } else if (f.steps() == o.max_subspace) {
        const auto ta = std::chrono::steady_clock::now();
        extract();
        const auto tb = std::chrono::steady_clock::now();
        t_extract += std::chrono::duration<double>(tb - ta).count();
        if (top_k_converged()) break;
        if (mvps + 2 > o.max_mvps) break;
        f.thick_restart(o.keep, &ritz);
        t_restart += std::chrono::duration<double>(std::chrono::steady_clock::now() - tb).count();
        ++out.restarts;
      }
      continue;
    }
    const StepInfo step = f.step(o, norm_scale, &mvps);
    if (step.status == 1) {
      ++out.deflations;
      ++consecutive_breakdowns;
      f.compress_exhausted();
      extract();
      if (top_k_converged() || consecutive_breakdowns > 3) break;
      f.deflate_right();
      continue;
    }
    ++out.steps;
    if (step.reorth_left) ++out.reorth_count;
    if (step.reorth_right) ++out.reorth_count;
    norm_scale = std::max(norm_scale, std::hypot(step.alpha, step.beta));
    if (step.status == 2) {
      ++out.deflations;
      ++consecutive_breakdowns;
    } else {
      consecutive_breakdowns = 0;
    }
    if (!o.thick) {
      extract();
      if (top_k_converged()) break;
    } else if (f.steps() == o.max_subspace) {
      extract();
      if (top_k_converged()) break;
      if (mvps + 2 > o.max_mvps) break;
      f.thick_restart(o.keep, &ritz);
      ++out.restarts;
    }
  }

  const auto t_loop = std::chrono::steady_clock::now();
  extract();
  const int64_t j = f.steps();
  const int64_t count = std::min<int64_t>(o.k, j);
  out.count = count;
  out.singvals.assign(ritz.values.begin(), ritz.values.begin() + count);
  out.err.assign(ritz.err.begin(), ritz.err.begin() + count);
  out.converged.assign(ritz.converged.begin(), ritz.converged.begin() + count);
  out.U.reset(new double[(size_t)std::max<int64_t>(m * count, 1)]);
  out.V.reset(new double[(size_t)std::max<int64_t>(n * count, 1)]);
  // Ritz vectors U W_L, V W_R, returned as-is (gkl.cpp:500-507).
  const auto t_ext = std::chrono::steady_clock::now();
  f.ritz_vectors(ritz, count, out.U.get(), out.V.get());
  const auto t_vec = std::chrono::steady_clock::now();
  out.all_converged = count == o.k && top_k_converged();
  out.mvps = mvps;
  ctx->set_device(0);
  GKB_CUDA(cudaEventRecord(e1, ctx->shards[0].stream));
  GKB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  GKB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out.device_seconds = ms * 1e-3;
  out.host_syncs = f.host_syncs;
  out.fused_tails = f.fused_tails;
  if (const char* e = getenv("GKB_VERBOSE"))
    if (e[0] == '1')
    {
      auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
      fprintf(stderr, "[gkb] svdl: %lld steps, host syncs %lld, speculative right half-steps kept %lld / "
              "not used %lld; loop %.4f s, final extract %.4f s, Ritz vectors %.4f s\n",
              (long long)out.steps, (long long)f.host_syncs, (long long)f.spec_hits,
              (long long)f.spec_misses, sec(t_start, t_loop), sec(t_loop, t_ext),
              sec(t_ext, t_vec));
      fprintf(stderr, "[gkb] svdl cycles: enqueue %.4f s, wait %.4f s, Ritz extract %.4f s, "
              "thick restart %.4f s\n", f.t_enqueue, f.t_wait, t_extract, t_restart);
    }
  op->mvps += mvps;
  out.wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return out;
}

}  // namespace gkb
