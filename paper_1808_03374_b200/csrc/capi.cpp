// extern "C" boundary (include/gkb.h). Converts C++ exceptions to status
// codes + a thread-local message; no exception crosses the ABI.
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "host.hpp"

struct gkb_ctx {
  gkb::Context c;
};
struct gkb_op {
  gkb_ctx* ctx;
  std::unique_ptr<gkb::DevOp> op;
  gkb::GenoOp* geno = nullptr;
};
struct gkb_lanczos {
  gkb_op* op;
  std::unique_ptr<gkb::Lanczos> lz;
};

namespace gkb {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace gkb

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return GKB_OK;
  } catch (const gkb::Error& e) {
    gkb::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    gkb::set_last_error("out of memory");
    return GKB_EOOM;
  } catch (const std::exception& e) {
    gkb::set_last_error(e.what());
    return GKB_ELOGIC;
  } catch (...) {
    gkb::set_last_error("unknown error");
    return GKB_ELOGIC;
  }
}

void need(const void* p, const char* what) {
  if (!p) gkb::fail(GKB_EINVAL, std::string(what) + " is null");
}

}  // namespace

extern "C" {

const char* gkb_last_error(void) { return gkb::g_last_error.c_str(); }
const char* gkb_version(void) { return "gkb 0.1.0 (sm_100a)"; }

int gkb_init(int nshards, const int* devices, gkb_ctx** ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    std::vector<int> devs;
    for (int i = 0; i < nshards; ++i) devs.push_back(devices ? devices[i] : 0);
    auto c = std::make_unique<gkb_ctx>();
    c->c.init_local(devs);
    *ctx = c.release();
  });
}

int gkb_nccl_unique_id(uint8_t id_out[128]) {
  return guarded([&] {
    need(id_out, "id_out");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) gkb::fail(GKB_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(id_out, &id, 128);
  });
}

int gkb_init_nccl(int device, const uint8_t id[128], int nranks, int rank, gkb_ctx** ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    need(id, "id");
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    auto c = std::make_unique<gkb_ctx>();
    c->c.init_nccl(device, uid, nranks, rank);
    *ctx = c.release();
  });
}

int gkb_init_host_comm(int device, int nranks, int rank, gkb_host_allreduce_fn fn, void* user,
                       gkb_ctx** ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    auto c = std::make_unique<gkb_ctx>();
    c->c.init_host(device, nranks, rank, fn, user);
    *ctx = c.release();
  });
}

int gkb_destroy(gkb_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int gkb_ctx_info(gkb_ctx* ctx, int* nloc, int* ntot, int* first) {
  return guarded([&] {
    need(ctx, "ctx");
    if (nloc) *nloc = (int)ctx->c.shards.size();
    if (ntot) *ntot = ctx->c.nshards_total;
    if (first) *first = ctx->c.first_shard;
  });
}

int gkb_synchronize(gkb_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->c.sync_all();
  });
}

int gkb_partition_rows(int64_t m, int nparts, int64_t* starts) {
  return guarded([&] {
    need(starts, "starts");
    const auto st = gkb::partition_rows(m, nparts);
    std::copy(st.begin(), st.end(), starts);
  });
}

int gkb_geno_from_bed(gkb_ctx* ctx, const uint8_t* payload, int64_t p, int64_t n, gkb_op** op) {
  return guarded([&] {
    need(ctx, "ctx");
    need(payload, "payload");
    need(op, "op");
    auto h = std::make_unique<gkb_op>();
    h->ctx = ctx;
    auto g = std::make_unique<gkb::GenoOp>();
    g->ctx = &ctx->c;
    g->build_from_payload(payload, p, n);
    h->geno = g.get();
    h->op = std::move(g);
    *op = h.release();
  });
}

int gkb_bed_check(const char* bed, const char* bim, const char* fam, int64_t* p, int64_t* n) {
  return guarded([&] {
    need(bed, "bed");
    need(bim, "bim");
    need(fam, "fam");
    need(p, "p");
    need(n, "n");
    gkb::bed_check(bed, bim, fam, p, n);
  });
}

int gkb_geno_from_bed_file(gkb_ctx* ctx, const char* bed, const char* bim, const char* fam,
                           gkb_op** op) {
  return guarded([&] {
    need(ctx, "ctx");
    need(bed, "bed");
    need(bim, "bim");
    need(fam, "fam");
    need(op, "op");
    int64_t p = 0, n = 0;
    gkb::bed_check(bed, bim, fam, &p, &n);
    auto h = std::make_unique<gkb_op>();
    h->ctx = ctx;
    auto g = std::make_unique<gkb::GenoOp>();
    g->ctx = &ctx->c;
    g->build_from_bed_file(bed, p, n);
    h->geno = g.get();
    h->op = std::move(g);
    *op = h.release();
  });
}

int gkb_geno_from_synth(gkb_ctx* ctx, const gkb_synth_spec* spec, gkb_op** op) {
  return guarded([&] {
    need(ctx, "ctx");
    need(spec, "spec");
    need(op, "op");
    auto h = std::make_unique<gkb_op>();
    h->ctx = ctx;
    auto g = std::make_unique<gkb::GenoOp>();
    g->ctx = &ctx->c;
    gkb::dev::SynthDev sd{};
    g->build_from_synth(sd, spec);
    h->geno = g.get();
    h->op = std::move(g);
    *op = h.release();
  });
}

static gkb::GenoOp* as_geno(gkb_op* op) {
  need(op, "op");
  if (!op->geno) gkb::fail(GKB_EINVAL, "operator is not a genotype operator");
  return op->geno;
}

int gkb_geno_counts(gkb_op* op, int64_t* counts) {
  return guarded([&] {
    auto* g = as_geno(op);
    need(counts, "counts");
    std::copy(g->counts_host.begin(), g->counts_host.end(), counts);
  });
}

int gkb_geno_marker_scan(gkb_op* op, const double* y, const double* Z, int64_t k, int unbiased,
                         double* beta, double* se, double* intercept, double* sigma2,
                         int32_t* dep) {
  return guarded([&] {
    auto* g = as_geno(op);
    need(y, "y");
    if (k < 0) gkb::fail(GKB_EINVAL, "marker_scan: k must be >= 0");
    if (k > 0) need(Z, "Z");
    need(beta, "beta");
    need(se, "se");
    need(intercept, "intercept");
    need(sigma2, "sigma2");
    need(dep, "dep");
    g->marker_scan(y, Z, k, unbiased != 0, beta, se, intercept, sigma2, dep);
  });
}

int gkb_geno_standardize(gkb_op* op, int scheme) {
  return guarded([&] {
    auto* g = as_geno(op);
    std::vector<double> mu((size_t)g->m), is((size_t)g->m);
    gkb::marker_scaling(g->counts_host.data(), g->m, g->n, scheme, mu.data(), is.data());
    g->set_scaling(mu.data(), is.data());
  });
}

int gkb_geno_set_scaling(gkb_op* op, const double* mu, const double* inv_s) {
  return guarded([&] {
    auto* g = as_geno(op);
    need(mu, "mu");
    need(inv_s, "inv_s");
    g->set_scaling(mu, inv_s);
  });
}

int gkb_geno_get_scaling(gkb_op* op, double* mu, double* inv_s) {
  return guarded([&] {
    auto* g = as_geno(op);
    need(mu, "mu");
    need(inv_s, "inv_s");
    g->get_scaling(mu, inv_s);
  });
}

int gkb_geno_read_bed(gkb_op* op, int64_t row0, int64_t nrows, uint8_t* out) {
  return guarded([&] {
    auto* g = as_geno(op);
    need(out, "out");
    g->read_bed(row0, nrows, out);
  });
}

int gkb_geno_info(gkb_op* op, int64_t* nmissing, int64_t* packed_bytes, int64_t* device_bytes) {
  return guarded([&] {
    auto* g = as_geno(op);
    int64_t nm = 0;
    for (const auto& s : g->gs) nm += s.nmissing;
    if (nmissing) *nmissing = nm;
    if (packed_bytes) *packed_bytes = g->packed_bytes();
    if (device_bytes) *device_bytes = g->device_bytes();
  });
}

int gkb_dense_create(gkb_ctx* ctx, const double* X, int64_t m, int64_t n, gkb_op** op) {
  return guarded([&] {
    need(ctx, "ctx");
    need(X, "X");
    need(op, "op");
    auto h = std::make_unique<gkb_op>();
    h->ctx = ctx;
    auto d = std::make_unique<gkb::DenseOp>();
    d->ctx = &ctx->c;
    d->build(X, m, n);
    h->op = std::move(d);
    *op = h.release();
  });
}

int gkb_op_shape(gkb_op* op, int64_t* rows, int64_t* cols) {
  return guarded([&] {
    need(op, "op");
    if (rows) *rows = op->op->m;
    if (cols) *cols = op->op->n;
  });
}

int gkb_op_apply(gkb_op* op, const double* x, double* y) {
  return guarded([&] {
    need(op, "op");
    need(x, "x");
    need(y, "y");
    op->op->apply_host(x, y);
    ++op->op->mvps;
  });
}

int gkb_host_alloc(size_t bytes, void** ptr) {
  return guarded([&] {
    need(ptr, "ptr");
    *ptr = nullptr;
    if (bytes == 0) gkb::fail(GKB_EINVAL, "host_alloc: zero bytes");
    GKB_CUDA(cudaMallocHost(ptr, bytes));
  });
}

int gkb_host_free(void* ptr) {
  return guarded([&] {
    if (ptr) GKB_CUDA(cudaFreeHost(ptr));
  });
}

int gkb_op_apply_adjoint(gkb_op* op, const double* x, double* y) {
  return guarded([&] {
    need(op, "op");
    need(x, "x");
    need(y, "y");
    op->op->adjoint_host(x, y);
    ++op->op->mvps;
  });
}

int64_t gkb_op_mvps(gkb_op* op) { return op ? op->op->mvps : -1; }

int gkb_op_destroy(gkb_op* op) {
  return guarded([&] {
    if (op) op->ctx->c.sync_all();
    delete op;
  });
}

int gkb_op_bench(gkb_op* op, int which, int iters, int flush_l2, double* ms_per_iter,
                 double* main_ms_per_iter, int* launches_per_iter) {
  return guarded([&] {
    need(op, "op");
    if (iters < 1) gkb::fail(GKB_EINVAL, "iters < 1");
    if (which < 0 || which > 3) gkb::fail(GKB_EINVAL, "which must be 0, 1, 2 or 3");
    gkb::Context& c = op->ctx->c;
    gkb::DevOp* d = op->op.get();
    const int L = (int)c.shards.size();
    // x: Rng(7).uniform_symmetric() normalized (the start-vector convention,
    // gkl.cpp:428-429); y = X x computed once and reused by the adjoint.
    std::vector<double> xh((size_t)d->n);
    gkb::Rng rng(7);
    double nrm = 0.0;
    for (auto& v : xh) {
      v = rng.uniform_symmetric();
      nrm += v * v;
    }
    nrm = std::sqrt(nrm);
    for (auto& v : xh) v /= nrm;
    std::vector<const double*> xi(L), yc(L);
    std::vector<double*> yi(L), zi(L);
    for (int i = 0; i < L; ++i) {
      c.set_device(i);
      gkb::Shard& s = c.shards[i];
      GKB_CUDA(cudaMemcpyAsync(d->xbuf[i], xh.data(), sizeof(double) * (size_t)d->n,
                               cudaMemcpyHostToDevice, s.stream));
      xi[i] = d->xbuf[i];
      yi[i] = d->ybuf[i];
      yc[i] = d->ybuf[i];
      zi[i] = d->zbuf[i];
      if (flush_l2 && !s.flush_buf) {
        s.flush_bytes = (size_t)256 << 20;  // 2x the 126 MB L2
        GKB_CUDA(cudaMalloc(&s.flush_buf, s.flush_bytes));
      }
    }
    d->apply_dev(xi, yi);
    c.sync_all();
    c.set_device(0);
    cudaStream_t st = c.shards[0].stream;
    cudaEvent_t e0, e1;
    GKB_CUDA(cudaEventCreate(&e0));
    GKB_CUDA(cudaEventCreate(&e1));
    auto flush_all = [&]() {
      for (int i = 0; i < L; ++i) {
        c.set_device(i);
        gkb::dev::flush_l2(c.shards[i].flush_buf, c.shards[i].flush_bytes, c.shards[i].stream);
      }
      c.set_device(0);
    };
    auto timed = [&](auto&& body) {
      c.sync_all();
      GKB_CUDA(cudaEventRecord(e0, st));
      for (int t = 0; t < iters; ++t) body();
      GKB_CUDA(cudaEventRecord(e1, st));
      GKB_CUDA(cudaEventSynchronize(e1));
      c.sync_all();
      float f = 0.f;
      GKB_CUDA(cudaEventElapsedTime(&f, e0, e1));
      return (double)f;
    };
    double flush_ms = 0.0;
    if (flush_l2) flush_ms = timed([&] { flush_all(); });
    // which 3: a two-column block of each product (operator block path)
    double *X2 = nullptr, *Y2 = nullptr, *Z2 = nullptr;
    if (which == 3) {
      if (L != 1) gkb::fail(GKB_EINVAL, "bench: which 3 needs a single shard");
      c.set_device(0);
      GKB_CUDA(cudaMalloc(&X2, sizeof(double) * (size_t)(2 * d->n)));
      GKB_CUDA(cudaMalloc(&Y2, sizeof(double) * (size_t)(2 * std::max<int64_t>(d->m, 1))));
      GKB_CUDA(cudaMalloc(&Z2, sizeof(double) * (size_t)(2 * d->n)));
      for (int q = 0; q < 2; ++q)
        GKB_CUDA(cudaMemcpyAsync(X2 + q * d->n, xh.data(), sizeof(double) * (size_t)d->n,
                                 cudaMemcpyHostToDevice, c.shards[0].stream));
    }
    // whole step: K1 (+reduce) and/or K2 (+reduce, +cross-shard sum)
    const double total = timed([&] {
      if (flush_l2) flush_all();
      if (which == 0 || which == 2) d->apply_dev(xi, yi);
      if (which == 1 || which == 2) d->adjoint_dev(yc, zi);
      if (which == 3) {
        d->apply_block_dev({X2}, d->n, 2, {Y2}, {d->m});
        d->adjoint_block_dev({Y2}, {d->m}, 2, {Z2}, d->n);
      }
    });
    if (X2) cudaFree(X2);
    if (Y2) cudaFree(Y2);
    if (Z2) cudaFree(Z2);
    GKB_LAUNCH_CHECK();
    if (ms_per_iter) *ms_per_iter = (total - flush_ms) / iters;
    double main_ms = 0.0;
    int launches = 0;
    if (op->geno && which == 3) {
      launches = 10 * L;  // per product pair: 2 digitize + 1 two-vector main + 2 reduce
    } else if (op->geno) {
      gkb::GenoShard& g = op->geno->gs[0];
      const double t = timed([&] {
        if (flush_l2) flush_all();
        if (which == 0 || which == 2) gkb::dev::k1_main_only(g.view(), xi[0], st);
        if (which == 1 || which == 2) gkb::dev::k2_main_only(g.view(), st);
      });
      GKB_LAUNCH_CHECK();
      main_ms = (t - flush_ms) / iters;
      launches = (which == 2 ? 6 : 3) * L;  // digitize + main + reduce per product
    } else {
      launches = (which == 2 ? 2 : 1) * L;
    }
    if (main_ms_per_iter) *main_ms_per_iter = main_ms;
    if (launches_per_iter) *launches_per_iter = launches;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

void gkb_gkl_options_default(gkb_gkl_options* o) {
  if (!o) return;
  o->k = 10;
  o->tol = 1e-8;
  o->max_mvps = 1000000;
  o->reorth = 1;
  o->omega = 1e-8;
  o->one_sided = 0;
  o->restart = 0;
  o->max_subspace = 40;
  o->keep = 20;
  o->seed = 0;
  o->record_history = 0;
  o->omega_recurrence = 1;
}

int gkb_gkl_options_validate(const gkb_gkl_options* o, int64_t m, int64_t n) {
  return guarded([&] {
    need(o, "options");
    gkb::validate_options(gkb::options_from(o), m, n);
  });
}

int gkb_svdl(gkb_op* op, const gkb_gkl_options* o, gkb_svdl_result** res) {
  return guarded([&] {
    need(op, "op");
    need(o, "options");
    need(res, "res");
    gkb::SvdlOutput out = gkb::svdl(op->op.get(), gkb::options_from(o));
    auto* r = new gkb_svdl_result();
    std::memset(r, 0, sizeof(*r));
    r->m = op->op->m;
    r->n = op->op->n;
    r->count = out.count;
    auto dup = [](const std::vector<double>& v) {
      double* p = new double[v.size() > 0 ? v.size() : 1];
      std::copy(v.begin(), v.end(), p);
      return p;
    };
    r->singvals = dup(out.singvals);
    r->U = out.U.release();  // new[] -> delete[] in gkb_svdl_result_free
    r->V = out.V.release();
    r->err_estimates = dup(out.err);
    r->converged = new int32_t[out.converged.size() > 0 ? out.converged.size() : 1];
    std::copy(out.converged.begin(), out.converged.end(), r->converged);
    r->mvps = out.mvps;
    r->steps = out.steps;
    r->restarts = out.restarts;
    r->reorth_count = out.reorth_count;
    r->deflations = out.deflations;
    r->all_converged = out.all_converged ? 1 : 0;
    r->wall_seconds = out.wall_seconds;
    r->history_len = out.history_len;
    r->ritz_history = dup(out.ritz_history);
    r->err_history = dup(out.err_history);
    r->device_seconds = out.device_seconds;
    r->host_syncs = out.host_syncs;
    r->fused_tails = out.fused_tails;
    *res = r;
  });
}

int gkb_subspace_qr(gkb_op* op, int64_t k, double tol, int64_t max_iter, uint64_t seed,
                    int scaled_delta, gkb_subspace_result** res) {
  return guarded([&] {
    need(op, "op");
    need(res, "res");
    gkb::SubspaceOutput o =
        gkb::subspace_qr_device(op->op.get(), k, tol, max_iter, seed, scaled_delta != 0);
    auto* r = new gkb_subspace_result();
    std::memset(r, 0, sizeof(*r));
    auto dup = [](const std::vector<double>& v) {
      double* p = new double[v.size() > 0 ? v.size() : 1];
      std::copy(v.begin(), v.end(), p);
      return p;
    };
    r->m = op->op->m;
    r->k = k;
    r->basis = dup(o.basis);
    r->eigvals = dup(o.eigvals);
    r->singvals = dup(o.singvals);
    r->iterations = o.iterations;
    r->delta_history = dup(o.delta_history);
    r->invcond_history = dup(o.invcond_history);
    r->converged = o.converged ? 1 : 0;
    r->rank_deficient = o.rank_deficient ? 1 : 0;
    r->mvps = o.mvps;
    *res = r;
  });
}

int gkb_subspace_result_free(gkb_subspace_result* r) {
  return guarded([&] {
    if (!r) return;
    for (double* p : {r->basis, r->eigvals, r->singvals, r->delta_history, r->invcond_history})
      delete[] p;
    delete r;
  });
}

int gkb_svdl_result_free(gkb_svdl_result* r) {
  return guarded([&] {
    if (!r) return;
    delete[] r->singvals;
    delete[] r->U;
    delete[] r->V;
    delete[] r->err_estimates;
    delete[] r->converged;
    delete[] r->ritz_history;
    delete[] r->err_history;
    delete r;
  });
}

int gkb_lanczos_create(gkb_op* op, int64_t capacity, const double* start, uint64_t rng_seed,
                       gkb_lanczos** lz) {
  return guarded([&] {
    need(op, "op");
    need(start, "start");
    need(lz, "lz");
    auto h = std::make_unique<gkb_lanczos>();
    h->op = op;
    h->lz = std::make_unique<gkb::Lanczos>(op->op.get(), capacity, start, rng_seed);
    *lz = h.release();
  });
}

int gkb_lanczos_destroy(gkb_lanczos* lz) {
  return guarded([&] { delete lz; });
}

int gkb_bidiag_step(gkb_lanczos* lz, const gkb_gkl_options* o, double norm_scale, int* status,
                    int* reorth_left, int* reorth_right, double* alpha, double* beta) {
  return guarded([&] {
    need(lz, "lz");
    need(o, "options");
    int64_t mv = 0;
    const gkb::StepInfo info = lz->lz->step(gkb::options_from(o), norm_scale, &mv);
    lz->op->op->mvps += mv;
    if (status) *status = info.status;
    if (reorth_left) *reorth_left = info.reorth_left;
    if (reorth_right) *reorth_right = info.reorth_right;
    if (alpha) *alpha = info.alpha;
    if (beta) *beta = info.beta;
  });
}

int gkb_lanczos_info(gkb_lanczos* lz, int64_t* steps, int64_t* capacity, int* right_exhausted) {
  return guarded([&] {
    need(lz, "lz");
    if (steps) *steps = lz->lz->steps();
    if (capacity) *capacity = lz->lz->capacity();
    if (right_exhausted) *right_exhausted = lz->lz->right_exhausted();
  });
}

int gkb_lanczos_get(gkb_lanczos* lz, double* U, double* V, double* B, double* coupling,
                    double* omega_left, double* omega_right) {
  return guarded([&] {
    need(lz, "lz");
    lz->lz->get(U, V, B, coupling, omega_left, omega_right);
  });
}

int gkb_ritz_extract(gkb_lanczos* lz, double tol, double* values, double* WL, double* WR,
                     double* err, double* err_crude, int32_t* converged) {
  return guarded([&] {
    need(lz, "lz");
    const gkb::Ritz r = lz->lz->ritz_extract(tol);
    if (values) std::copy(r.values.begin(), r.values.end(), values);
    if (WL) std::copy(r.WL.begin(), r.WL.end(), WL);
    if (WR) std::copy(r.WR.begin(), r.WR.end(), WR);
    if (err) std::copy(r.err.begin(), r.err.end(), err);
    if (err_crude) std::copy(r.err_crude.begin(), r.err_crude.end(), err_crude);
    if (converged) std::copy(r.converged.begin(), r.converged.end(), converged);
  });
}

int gkb_thick_restart(gkb_lanczos* lz, int64_t keep) {
  return guarded([&] {
    need(lz, "lz");
    lz->lz->thick_restart(keep);
  });
}

int gkb_compress_exhausted(gkb_lanczos* lz) {
  return guarded([&] {
    need(lz, "lz");
    lz->lz->compress_exhausted();
  });
}

int gkb_geno_plan(int64_t p_loc, int64_t n, double missing_fraction, int64_t free_bytes,
                  int* layouts, int64_t* dual_bytes, int64_t* single_bytes) {
  return guarded([&] {
    if (p_loc < 0 || n < 0) gkb::fail(GKB_EINVAL, "gkb_geno_plan: negative size");
    const gkb::LayoutPlan pl = gkb::plan_layouts(p_loc, n, missing_fraction, free_bytes);
    if (layouts) *layouts = pl.layouts;
    if (dual_bytes) *dual_bytes = pl.dual_bytes;
    if (single_bytes) *single_bytes = pl.single_bytes;
  });
}

int gkb_geno_layouts(gkb_op* op, int* layouts, int* dense_missing) {
  return guarded([&] {
    auto* g = as_geno(op);
    int l = 2, d = 0;
    for (const auto& sh : g->gs) {
      if (sh.single) l = 1;
      if (sh.ind) d = 1;
    }
    if (layouts) *layouts = l;
    if (dense_missing) *dense_missing = d;
  });
}

int gkb_deflate_right(gkb_lanczos* lz) {
  return guarded([&] {
    need(lz, "lz");
    lz->lz->deflate_right();
  });
}

int gkb_cgs2(gkb_ctx* ctx, const double* basis, int64_t len, int64_t ncols, double* v,
             double* coeffs, double* norm_after) {
  return guarded([&] {
    need(ctx, "ctx");
    need(v, "v");
    if (ncols > 0) need(basis, "basis");
    gkb::Context& c = ctx->c;
    c.set_device(0);
    gkb::Shard& s = c.shards[0];
    if (len < 0 || ncols < 0) gkb::fail(GKB_EINVAL, "cgs2: negative size");
    // result slots: ncols + 3 (first pass) + ncols + 2 (second pass)
    s.ensure_res(2 * ncols + 8);
    gkb::DevScratch Qh, dvh;
    GKB_CUDA(cudaMalloc(&Qh.p, sizeof(double) * (size_t)std::max<int64_t>(len * ncols, 1)));
    GKB_CUDA(cudaMalloc(&dvh.p, sizeof(double) * (size_t)std::max<int64_t>(len, 1)));
    double* Q = Qh.as<double>();
    double* dv = dvh.as<double>();
    if (ncols > 0)
      GKB_CUDA(cudaMemcpyAsync(Q, basis, sizeof(double) * (size_t)(len * ncols),
                               cudaMemcpyHostToDevice, s.stream));
    GKB_CUDA(cudaMemcpyAsync(dv, v, sizeof(double) * (size_t)len, cudaMemcpyHostToDevice,
                             s.stream));
    s.ensure_partial(gkb::dev::red_blocks(len) * (ncols + 4) + 64);
    const double eta = 0.70710678118654752440;
    double na;
    std::vector<double> cf((size_t)std::max<int64_t>(ncols, 1), 0.0);
    if (ncols == 0) {
      gkb::dev::nrm2sq(dv, len, s.rs, s.dres, s.stream);
      GKB_CUDA(cudaMemcpyAsync(s.hres, s.dres, 8, cudaMemcpyDeviceToHost, s.stream));
      GKB_CUDA(cudaStreamSynchronize(s.stream));
      na = std::sqrt(s.hres[0]);
    } else {
      gkb::dev::gemv_t(Q, len, len, ncols, dv, true, s.rs, s.dres, s.stream);
      gkb::dev::gemv_n(Q, len, len, ncols, s.dres, dv, 1.0, -1.0, true, s.rs, s.dres + ncols + 1,
                       s.stream);
      GKB_CUDA(cudaMemcpyAsync(s.hres, s.dres, sizeof(double) * (size_t)(ncols + 3),
                               cudaMemcpyDeviceToHost, s.stream));
      GKB_CUDA(cudaStreamSynchronize(s.stream));
      const double nb = std::sqrt(s.hres[ncols]);
      na = std::sqrt(s.hres[ncols + 2]);
      for (int64_t i = 0; i < ncols; ++i) cf[i] = s.hres[i];
      if (na < eta * nb) {
        const int64_t o = ncols + 3;
        gkb::dev::gemv_t(Q, len, len, ncols, dv, false, s.rs, s.dres + o, s.stream);
        gkb::dev::gemv_n(Q, len, len, ncols, s.dres + o, dv, 1.0, -1.0, true, s.rs,
                         s.dres + o + ncols, s.stream);
        GKB_CUDA(cudaMemcpyAsync(s.hres, s.dres, sizeof(double) * (size_t)(o + ncols + 2),
                                 cudaMemcpyDeviceToHost, s.stream));
        GKB_CUDA(cudaStreamSynchronize(s.stream));
        for (int64_t i = 0; i < ncols; ++i) cf[i] += s.hres[o + i];
        na = std::sqrt(s.hres[o + ncols + 1]);
      }
    }
    GKB_LAUNCH_CHECK();
    GKB_CUDA(cudaMemcpyAsync(v, dv, sizeof(double) * (size_t)len, cudaMemcpyDeviceToHost,
                             s.stream));
    GKB_CUDA(cudaStreamSynchronize(s.stream));
    if (coeffs)
      for (int64_t i = 0; i < ncols; ++i) coeffs[i] += cf[i];
    if (norm_after) *norm_after = na;
  });
}

int gkb_svd_small(const double* M, int64_t r, int64_t c, double* U, double* s, double* V) {
  return guarded([&] {
    need(M, "M");
    gkb::svd_small(M, r, c, U, s, V);
  });
}

int gkb_rng_fill_normal(uint64_t seed, int64_t n, double* out) {
  return guarded([&] {
    need(out, "out");
    gkb::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
  });
}

int gkb_op_apply_block(gkb_op* op, const double* X, int64_t k, double* Y) {
  return guarded([&] {
    need(op, "op");
    need(X, "X");
    need(Y, "Y");
    if (k < 0) gkb::fail(GKB_EINVAL, "apply_block: k must be >= 0");
    if (k == 0) return;
    op->op->apply_block_host(X, k, Y);
    op->op->mvps += k;
  });
}

int gkb_op_apply_adjoint_block(gkb_op* op, const double* Y, int64_t k, double* Z) {
  return guarded([&] {
    need(op, "op");
    need(Y, "Y");
    need(Z, "Z");
    if (k < 0) gkb::fail(GKB_EINVAL, "apply_adjoint_block: k must be >= 0");
    if (k == 0) return;
    op->op->adjoint_block_host(Y, k, Z);
    op->op->mvps += k;
  });
}

int gkb_rng_fill_symmetric(uint64_t seed, int64_t n, double* out) {
  return guarded([&] {
    need(out, "out");
    gkb::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform_symmetric();
  });
}

int gkb_marker_scaling(const int64_t* counts, int64_t p, int64_t n, int scheme, double* mu,
                       double* inv_s) {
  return guarded([&] {
    need(counts, "counts");
    need(mu, "mu");
    need(inv_s, "inv_s");
    gkb::marker_scaling(counts, p, n, scheme, mu, inv_s);
  });
}

}  // extern "C"
