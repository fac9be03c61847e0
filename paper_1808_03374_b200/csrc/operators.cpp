// Device operators: the packed genotype operator (replacing the reference's
// DenseOperator over the imputed, standardized matrix) and a device
// DenseOperator (linop.hpp:43-64). Rows (reference markers) are sharded;
// columns (samples) are replicated.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "host.hpp"

namespace gkb {

// ---------------------------------------------------------------- DevOp
DevOp::~DevOp() {
  for (size_t i = 0; i < xbuf.size(); ++i) {
    cudaSetDevice(ctx->shards[i].dev);
    cudaFree(xbuf[i]);
    cudaFree(ybuf[i]);
    cudaFree(zbuf[i]);
    if (i < yfull.size()) cudaFree(yfull[i]);
    if (i < bin_.size() && bin_[i]) cudaFree(bin_[i]);
    if (i < bout_.size() && bout_[i]) cudaFree(bout_[i]);
  }
}

void DevOp::alloc_host_api_buffers() {
  const int L = (int)ctx->shards.size();
  xbuf.assign(L, nullptr);
  ybuf.assign(L, nullptr);
  zbuf.assign(L, nullptr);
  yfull.assign(L, nullptr);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    GKB_CUDA(cudaMalloc(&xbuf[i], sizeof(double) * (size_t)std::max<int64_t>(n, 1)));
    GKB_CUDA(cudaMalloc(&ybuf[i], sizeof(double) * (size_t)std::max<int64_t>(rows(i), 1)));
    GKB_CUDA(cudaMalloc(&zbuf[i], sizeof(double) * (size_t)std::max<int64_t>(n, 1)));
    if (ctx->spmd_mode && ctx->nshards_total > 1)
      GKB_CUDA(cudaMalloc(&yfull[i], sizeof(double) * (size_t)std::max<int64_t>(m, 1)));
  }
}

// Page-locked host memory (cudaMallocHost, gkb_host_alloc / pinned_empty) is
// mapped into the device address space at the same address (UVA).
static bool device_accessible(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

// One local shard (no cross-shard sum) and an operator whose result kernels
// write each element once: page-locked host buffers are used in place.
bool DevOp::direct_io(const void* a, const void* b) const {
  if (!direct_host_io || ctx->shards.size() != 1 || (ctx->spmd_mode && ctx->nshards_total > 1))
    return false;
  return device_accessible(a) && (!b || device_accessible(b));
}

void DevOp::apply_host(const double* x, double* y) {
  const int L = (int)ctx->shards.size();
  if (direct_io(y, nullptr)) {  // y written by the reduce kernel over PCIe, no D2H copy
    ctx->set_device(0);
    GKB_CUDA(cudaMemcpyAsync(xbuf[0], x, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice,
                             ctx->shards[0].stream));
    host_out_ = true;
    try {
      apply_dev({xbuf[0]}, {y});
    } catch (...) {
      host_out_ = false;
      throw;
    }
    host_out_ = false;
    ctx->sync_all();
    return;
  }
  std::vector<const double*> xi(L);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    GKB_CUDA(cudaMemcpyAsync(xbuf[i], x, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice,
                             ctx->shards[i].stream));
    xi[i] = xbuf[i];
  }
  apply_dev(xi, ybuf);
  if (ctx->spmd_mode && ctx->nshards_total > 1) {
    Shard& s = ctx->shards[0];
    GKB_CUDA(cudaSetDevice(s.dev));
    GKB_CUDA(cudaMemsetAsync(yfull[0], 0, sizeof(double) * (size_t)m, s.stream));
    GKB_CUDA(cudaMemcpyAsync(yfull[0] + row0(0), ybuf[0], sizeof(double) * (size_t)rows(0),
                             cudaMemcpyDeviceToDevice, s.stream));
    ctx->allreduce({yfull[0]}, m);
    GKB_CUDA(cudaMemcpyAsync(y, yfull[0], sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost,
                             s.stream));
  } else {
    for (int i = 0; i < L; ++i) {
      ctx->set_device(i);
      GKB_CUDA(cudaMemcpyAsync(y + row0(i), ybuf[i], sizeof(double) * (size_t)rows(i),
                               cudaMemcpyDeviceToHost, ctx->shards[i].stream));
    }
  }
  ctx->sync_all();
}

void DevOp::adjoint_host(const double* y, double* z) {
  const int L = (int)ctx->shards.size();
  if (direct_io(y, z)) {  // y read once by digitize, z written by the reduce kernel
    ctx->set_device(0);
    adjoint_dev({y}, {z});
    ctx->sync_all();
    return;
  }
  std::vector<const double*> yi(L);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    GKB_CUDA(cudaMemcpyAsync(ybuf[i], y + row0(i), sizeof(double) * (size_t)rows(i),
                             cudaMemcpyHostToDevice, ctx->shards[i].stream));
    yi[i] = ybuf[i];
  }
  adjoint_dev(yi, zbuf);
  ctx->set_device(0);
  GKB_CUDA(cudaMemcpyAsync(z, zbuf[0], sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost,
                           ctx->shards[0].stream));
  ctx->sync_all();
}

void DevOp::ensure_block_buffers(int64_t in_doubles, int64_t out_doubles) {
  const int L = (int)ctx->shards.size();
  if ((int64_t)bin_.size() != L) {
    bin_.assign(L, nullptr);
    bout_.assign(L, nullptr);
    bin_cap_ = bout_cap_ = 0;
  }
  if (in_doubles > bin_cap_ || out_doubles > bout_cap_) {
    ctx->sync_all();
    const int64_t ci = std::max(in_doubles, bin_cap_), co = std::max(out_doubles, bout_cap_);
    for (int i = 0; i < L; ++i) {
      ctx->set_device(i);
      if (bin_[i]) cudaFree(bin_[i]);
      if (bout_[i]) cudaFree(bout_[i]);
      GKB_CUDA(cudaMalloc(&bin_[i], sizeof(double) * (size_t)std::max<int64_t>(ci, 1)));
      GKB_CUDA(cudaMalloc(&bout_[i], sizeof(double) * (size_t)std::max<int64_t>(co, 1)));
    }
    bin_cap_ = ci;
    bout_cap_ = co;
  }
}

void DevOp::apply_block_dev(const std::vector<const double*>& X, int64_t ldx, int64_t k,
                            const std::vector<double*>& Y, const std::vector<int64_t>& ldy) {
  const int L = (int)ctx->shards.size();
  for (int64_t c = 0; c < k; ++c) {
    std::vector<const double*> xi(L);
    std::vector<double*> yi(L);
    for (int i = 0; i < L; ++i) {
      xi[i] = X[i] + c * ldx;
      yi[i] = Y[i] + c * ldy[i];
    }
    apply_dev(xi, yi);
  }
}

void DevOp::adjoint_block_dev(const std::vector<const double*>& Yb,
                              const std::vector<int64_t>& ldyb, int64_t k,
                              const std::vector<double*>& Z, int64_t ldz) {
  const int L = (int)ctx->shards.size();
  for (int64_t c = 0; c < k; ++c) {
    std::vector<const double*> yi(L);
    std::vector<double*> zi(L);
    for (int i = 0; i < L; ++i) {
      yi[i] = Yb[i] + c * ldyb[i];
      zi[i] = Z[i] + c * ldz;
    }
    adjoint_dev(yi, zi);
  }
}

void DevOp::apply_block_host(const double* X, int64_t k, double* Y) {
  const int L = (int)ctx->shards.size();
  const bool spmd = ctx->spmd_mode && ctx->nshards_total > 1;
  int64_t rmax = 1;
  for (int i = 0; i < L; ++i) rmax = std::max(rmax, rows(i));
  // SPMD: every rank assembles the full m x k block for one allreduce;
  // local shards: each holds its own rows x k
  ensure_block_buffers(n * k, (spmd ? m : rmax) * k);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    GKB_CUDA(cudaMemcpyAsync(bin_[i], X, sizeof(double) * (size_t)(n * k), cudaMemcpyHostToDevice,
                             ctx->shards[i].stream));
  }
  {
    std::vector<const double*> xb(L);
    std::vector<double*> yb(L);
    std::vector<int64_t> ld(L);
    for (int i = 0; i < L; ++i) {
      xb[i] = bin_[i];
      yb[i] = spmd ? bout_[i] + row0(i) : bout_[i];
      ld[i] = spmd ? m : rows(i);
    }
    apply_block_dev(xb, n, k, yb, ld);
  }
  if (spmd) {
    // zero the other ranks' rows of every column, then one allreduce of m*k
    Shard& s = ctx->shards[0];
    ctx->set_device(0);
    const int64_t r0 = row0(0), r = rows(0);
    for (int64_t c = 0; c < k; ++c) {
      if (r0 > 0)
        GKB_CUDA(cudaMemsetAsync(bout_[0] + c * m, 0, sizeof(double) * (size_t)r0, s.stream));
      if (r0 + r < m)
        GKB_CUDA(cudaMemsetAsync(bout_[0] + c * m + r0 + r, 0, sizeof(double) * (size_t)(m - r0 - r),
                                 s.stream));
    }
    ctx->allreduce({bout_[0]}, m * k);
    GKB_CUDA(cudaMemcpyAsync(Y, bout_[0], sizeof(double) * (size_t)(m * k), cudaMemcpyDeviceToHost,
                             s.stream));
  } else {
    for (int i = 0; i < L; ++i) {
      ctx->set_device(i);
      if (rows(i) == 0) continue;
      GKB_CUDA(cudaMemcpy2DAsync(Y + row0(i), sizeof(double) * (size_t)m, bout_[i],
                                 sizeof(double) * (size_t)rows(i), sizeof(double) * (size_t)rows(i),
                                 (size_t)k, cudaMemcpyDeviceToHost, ctx->shards[i].stream));
    }
  }
  ctx->sync_all();
}

void DevOp::adjoint_block_host(const double* Yh, int64_t k, double* Z) {
  const int L = (int)ctx->shards.size();
  int64_t rmax = 1;
  for (int i = 0; i < L; ++i) rmax = std::max(rmax, rows(i));
  ensure_block_buffers(rmax * k, n * k);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    if (rows(i) == 0) continue;
    GKB_CUDA(cudaMemcpy2DAsync(bin_[i], sizeof(double) * (size_t)rows(i), Yh + row0(i),
                               sizeof(double) * (size_t)m, sizeof(double) * (size_t)rows(i),
                               (size_t)k, cudaMemcpyHostToDevice, ctx->shards[i].stream));
  }
  {
    std::vector<const double*> yb(L);
    std::vector<double*> zb(L);
    std::vector<int64_t> ld(L);
    for (int i = 0; i < L; ++i) {
      yb[i] = bin_[i];
      zb[i] = bout_[i];
      ld[i] = rows(i);
    }
    adjoint_block_dev(yb, ld, k, zb, n);
  }
  ctx->set_device(0);
  GKB_CUDA(cudaMemcpyAsync(Z, bout_[0], sizeof(double) * (size_t)(n * k), cudaMemcpyDeviceToHost,
                           ctx->shards[0].stream));
  ctx->sync_all();
}

// ---------------------------------------------------------------- scaling
// impute_mean + standardize (genio.cpp:124-185) restated on marker counts;
// identical formulas to the oracle's orc_marker_scaling (compiled without
// FMA contraction on both sides, so the results match bit for bit).
void marker_scaling(const int64_t* counts, int64_t p, int64_t n, int scheme, double* mu,
                    double* inv_s) {
  if (scheme < 0 || scheme > 3) fail(GKB_EINVAL, "standardize: unknown scaling scheme");
  if (n <= 0) fail(GKB_EINVAL, "standardize: no samples");  // genio.cpp:154
  const double nd = (double)n;
  for (int64_t j = 0; j < p; ++j) {
    const int64_t n0 = counts[4 * j], n1 = counts[4 * j + 1], n2 = counts[4 * j + 2];
    const int64_t obs = n0 + n1 + n2;
    if (scheme == 3) {
      mu[j] = 0.0;
      inv_s[j] = 1.0;
      continue;
    }
    const double mean = obs > 0 ? (double)(n1 + 2 * n2) / (double)obs : 0.0;
    mu[j] = mean;
    const int distinct = (n0 > 0) + (n1 > 0) + (n2 > 0);
    if (distinct < 2) {  // zero variance: zero row, flagged (genio.cpp:167-171)
      inv_s[j] = 0.0;
      continue;
    }
    double s;
    if (scheme == 0) {
      const double a = 0.0 - mean, b = 1.0 - mean, c = 2.0 - mean;
      const double ss = (double)n0 * (a * a) + (double)n1 * (b * b) + (double)n2 * (c * c);
      s = std::sqrt(ss / nd);
    } else if (scheme == 1) {
      const double clamp = 1.0 / (2.0 * nd + 2.0);
      double q = mean / 2.0;
      if (q < clamp) q = clamp;
      if (q > 1.0 - clamp) q = 1.0 - clamp;
      s = std::sqrt(q * (1.0 - q));
    } else {
      const double f = mean / 2.0;
      s = std::sqrt(2.0 * f * (1.0 - f));
    }
    inv_s[j] = s > 0.0 ? 1.0 / s : 0.0;
  }
}

// ---------------------------------------------------------------- GenoOp
// Per-CTA missing lists of one layout: count pass, per-block scan on device,
// block bases scanned on the host (nblk values), fill pass. Returns the number
// of entries (== the shard's missing count).
static int64_t build_block_lists(const uint32_t* lay, const dev::PMPlan& pl, cudaStream_t st,
                                 uint32_t** off, int64_t** base, uint16_t** ent, int64_t* bytes) {
  const int span = pl.rows_cta;
  const int64_t nblk = pl.grid_x * pl.nkc;
  uint32_t* cnt = nullptr;
  int64_t* tot = nullptr;
  auto pool = [&](auto** ptr, size_t bytes) {  // stream-ordered (no device sync)
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, st));
  };
  pool(&cnt, sizeof(uint32_t) * (size_t)(nblk * span));
  pool(&tot, sizeof(int64_t) * (size_t)nblk);
  // + 4: the main kernels bulk-copy a 16-byte-aligned superset of a block's offsets
  pool(off, sizeof(uint32_t) * (size_t)(nblk * (span + 1) + 4));
  dev::miss_lists(lay, pl, false, cnt, nullptr, nullptr, nullptr, st);
  GKB_LAUNCH_CHECK();
  dev::block_scan(cnt, nblk, span, *off, tot, st);
  GKB_LAUNCH_CHECK();
  std::vector<int64_t> h((size_t)nblk);
  GKB_CUDA(cudaMemcpyAsync(h.data(), tot, sizeof(int64_t) * (size_t)nblk, cudaMemcpyDeviceToHost, st));
  GKB_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(tot, st);
  int64_t total = 0;
  for (int64_t bb = 0; bb < nblk; ++bb) {
    const int64_t c = h[bb];
    h[bb] = total;
    total += c;
  }
  pool(base, sizeof(int64_t) * (size_t)nblk);
  GKB_CUDA(cudaMemcpyAsync(*base, h.data(), sizeof(int64_t) * (size_t)nblk, cudaMemcpyHostToDevice,
                           st));
  // padded to whole 16-byte chunks plus one: the main kernels stage a run with
  // 16-byte cp.async copies whose end is rounded up (tail zeroed, never used)
  const int64_t ent_alloc = (total + 7) / 8 * 8 + 8;
  pool(ent, sizeof(uint16_t) * (size_t)ent_alloc);
  GKB_CUDA(cudaMemsetAsync(*ent + total, 0, sizeof(uint16_t) * (size_t)(ent_alloc - total), st));
  dev::miss_lists(lay, pl, true, nullptr, *off, *base, *ent, st);
  GKB_LAUNCH_CHECK();
  *bytes += (int64_t)(sizeof(uint32_t) * nblk * (span + 1) + sizeof(int64_t) * nblk +
                      sizeof(uint16_t) * total);
  return total;
}

// Missing lists of the single-layout K2 blocks (1024 samples x 1792 SNPs,
// dev::miss_lists_l1t), into the shard's m2 fields. Returns the entry count.
static int64_t build_l1t_lists(GenoShard& g, cudaStream_t st) {
  const dev::L1TPlan& lt = g.plt;
  const int span = 1024;
  const int64_t nblk = lt.grid_x * lt.nkc;
  uint32_t* cnt = nullptr;
  int64_t* tot = nullptr;
  auto pool = [&](auto** ptr, size_t bytes) {
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, st));
  };
  pool(&cnt, sizeof(uint32_t) * (size_t)(nblk * span));
  pool(&tot, sizeof(int64_t) * (size_t)nblk);
  pool(&g.m2_off, sizeof(uint32_t) * (size_t)(nblk * (span + 1) + 4));
  dev::miss_lists_l1t(g.lt1, g.pl1, lt, g.p_loc, g.n, false, cnt, nullptr, nullptr, nullptr, st);
  GKB_LAUNCH_CHECK();
  dev::block_scan_1024(cnt, nblk, g.m2_off, tot, st);
  GKB_LAUNCH_CHECK();
  std::vector<int64_t> h((size_t)nblk);
  GKB_CUDA(cudaMemcpyAsync(h.data(), tot, sizeof(int64_t) * (size_t)nblk, cudaMemcpyDeviceToHost, st));
  GKB_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(tot, st);
  int64_t total = 0;
  for (int64_t bb = 0; bb < nblk; ++bb) {
    const int64_t c = h[bb];
    h[bb] = total;
    total += c;
  }
  pool(&g.m2_base, sizeof(int64_t) * (size_t)nblk);
  GKB_CUDA(cudaMemcpyAsync(g.m2_base, h.data(), sizeof(int64_t) * (size_t)nblk,
                           cudaMemcpyHostToDevice, st));
  const int64_t ent_alloc = (total + 7) / 8 * 8 + 8;
  pool(&g.m2_ent, sizeof(uint16_t) * (size_t)ent_alloc);
  GKB_CUDA(cudaMemsetAsync(g.m2_ent + total, 0, sizeof(uint16_t) * (size_t)(ent_alloc - total), st));
  dev::miss_lists_l1t(g.lt1, g.pl1, lt, g.p_loc, g.n, true, nullptr, g.m2_off, g.m2_base, g.m2_ent,
                      st);
  GKB_LAUNCH_CHECK();
  g.list_bytes += (int64_t)(sizeof(uint32_t) * nblk * (span + 1) + sizeof(int64_t) * nblk +
                            sizeof(uint16_t) * total);
  return total;
}

static void alloc_scratch(const dev::PMPlan& pl, bool with_cm, dev::PMScratch& sc,
                          cudaStream_t st) {
  auto pool = [&](auto** ptr, size_t bytes) {
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, st));
  };
  pool(&sc.dig, sizeof(uint4) * (size_t)(pl.nkc * pl.kt_cta * 64));
  pool(&sc.dexp, sizeof(int) * (size_t)pl.nkc);
  pool(&sc.dsum, sizeof(double) * (size_t)pl.nkc);
  pool(&sc.part, sizeof(double) * (size_t)(pl.nkc * pl.rows_pad));
  if (with_cm) pool(&sc.cm, sizeof(double) * (size_t)std::max<int64_t>(pl.C, 1));
  pool(&sc.tick, sizeof(unsigned) * (size_t)std::max<int64_t>(pl.grid_x, 1));
  GKB_CUDA(cudaMemsetAsync(sc.tick, 0, sizeof(unsigned) * (size_t)std::max<int64_t>(pl.grid_x, 1), st));
}

static void free_scratch(dev::PMScratch& sc, cudaStream_t st) {
  void* ptrs[] = {sc.dig, sc.dexp, sc.dsum, sc.part, sc.cm, sc.tick};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, st);
  sc = dev::PMScratch{};
}

dev::GenoView GenoShard::view() const {
  dev::GenoView v;
  v.lt1 = reinterpret_cast<const uint4*>(lt1);
  v.lt2 = reinterpret_cast<const uint4*>(lt2);
  v.pl1 = pl1;
  v.pl2 = pl2;
  v.p_loc = p_loc;
  v.n = n;
  v.mu = mu;
  v.mean = mean;
  v.inv_s = inv_s;
  const bool lists = nmissing > 0;
  v.m1 = dev::MissLists{lists ? m1_off : nullptr, m1_base, m1_ent};
  v.m2 = dev::MissLists{lists ? m2_off : nullptr, m2_base, m2_ent};
  v.s1 = s1;
  v.s2 = s2;
  v.nmissing = nmissing;
  v.ind = ind;
  v.s2m = s2m;
  v.single = single;
  v.l1t_grid = plt.grid_x;
  v.l1t_nkc = plt.nkc;
  v.l1t_rows_pad = plt.rows_pad;
  return v;
}

GenoOp::~GenoOp() {
  for (size_t i = 0; i < gs.size(); ++i) {
    cudaSetDevice(ctx->shards[i].dev);
    GenoShard& g = gs[i];
    cudaStream_t st = ctx->shards[i].stream;
    if (g.lt1) cudaFreeAsync(g.lt1, st);  // back to the pool (cudaMallocAsync)
    if (g.lt2) cudaFreeAsync(g.lt2, st);
    void* ptrs[] = {g.mu, g.mean, g.inv_s, g.counts, g.m1_off, g.m1_base, g.m1_ent, g.m2_off,
                    g.m2_base, g.m2_ent};
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, st);
    free_scratch(g.s1, st);
    free_scratch(g.s2, st);
    free_scratch(g.s1b, st);
    free_scratch(g.s2b, st);
    free_scratch(g.s2m, st);
    for (dev::TcScratch* t : {&g.tc1, &g.tc2}) {
      void* tp[] = {t->dig, t->dig2, t->dexp, t->dexp2, t->dsum, t->part};
      for (void* p : tp)
        if (p) cudaFreeAsync(p, st);
    }
    cudaStreamSynchronize(st);
  }
}

LayoutPlan plan_layouts(int64_t p_loc, int64_t n, double missing_fraction, int64_t free_bytes) {
  const dev::PMPlan pl1 = dev::pm_plan(p_loc, n), pl2 = dev::pm_plan(n, p_loc);
  const dev::L1TPlan lt = dev::l1t_plan(pl1, p_loc);
  const double nm = std::max(0.0, missing_fraction) * (double)p_loc * (double)n;
  auto lists = [&](int64_t blocks, int64_t span) {  // 16-bit entries + offsets + bases
    return (int64_t)(2.0 * nm) + blocks * ((span + 1) * 4 + 8);
  };
  const int64_t lay1 = 4 * dev::pm_words(pl1), lay2 = 4 * dev::pm_words(pl2);
  const int64_t l1 = lists(pl1.grid_x * pl1.nkc, 256), l2 = lists(pl2.grid_x * pl2.nkc, 256);
  const int64_t l2t = lists(lt.grid_x * lt.nkc, 1024);
  const int64_t part1 = 8 * pl1.nkc * pl1.rows_pad, part2 = 8 * pl2.nkc * pl2.rows_pad;
  const int64_t part2t = 8 * lt.nkc * lt.rows_pad;
  const int64_t vecs = 8 * 3 * pl1.rows_pad + 8 * (int64_t)(n + p_loc) * 8;
  // svdl's double-buffered bases at a 64-vector subspace
  const int64_t solver = 2 * 8 * 65 * (p_loc + n);
  LayoutPlan pl;
  pl.dual_bytes = lay1 + lay2 + l1 + l2 + part1 + part2 + vecs + solver;
  pl.single_bytes = lay1 + l1 + l2t + part1 + part2t + vecs + solver;
  pl.layouts = pl.dual_bytes <= free_bytes ? 2 : 1;
  return pl;
}

void GenoOp::alloc_shard(int i, int64_t p_loc, int64_t nn) {
  GenoShard& g = gs[i];
  g.p_loc = p_loc;
  g.n = nn;
  g.pl1 = dev::pm_plan(p_loc, nn);
  g.pl2 = dev::pm_plan(nn, p_loc);
  g.plt = dev::l1t_plan(g.pl1, p_loc);
  ctx->set_device(i);
  cudaStream_t st = ctx->shards[i].stream;
  {  // one layout or two (GKB_LAYOUTS=1|2 forces; else the device-memory plan)
    const char* e = std::getenv("GKB_LAYOUTS");
    if (e && std::strcmp(e, "1") == 0) {
      g.single = true;
    } else if (e && std::strcmp(e, "2") == 0) {
      g.single = false;
    } else {
      size_t fr = 0, tot = 0;
      GKB_CUDA(cudaMemGetInfo(&fr, &tot));
      const int64_t margin = (int64_t)2 << 30;
      g.single = plan_layouts(p_loc, nn, plan_missing, (int64_t)fr - margin).layouts == 1;
    }
  }
  const size_t w1 = (size_t)dev::pm_words(g.pl1), w2 = (size_t)dev::pm_words(g.pl2);
  // the two layouts are the large allocations: stream-ordered from the pool
  GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&g.lt1), sizeof(uint32_t) * w1, st));
  GKB_CUDA(cudaMemsetAsync(g.lt1, 0, sizeof(uint32_t) * w1, st));
  if (!g.single) {
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&g.lt2), sizeof(uint32_t) * w2, st));
    GKB_CUDA(cudaMemsetAsync(g.lt2, 0, sizeof(uint32_t) * w2, st));
  }
  const size_t pp = (size_t)g.pl1.rows_pad;
  // everything else too: no implicit device synchronization during ingest
  auto pool = [&](auto** ptr, size_t bytes) {
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, st));
  };
  pool(&g.mu, sizeof(double) * pp);
  pool(&g.mean, sizeof(double) * pp);
  pool(&g.inv_s, sizeof(double) * pp);
  GKB_CUDA(cudaMemsetAsync(g.mean, 0, sizeof(double) * pp, st));
  GKB_CUDA(cudaMemsetAsync(g.mu, 0, sizeof(double) * pp, st));
  GKB_CUDA(cudaMemsetAsync(g.inv_s, 0, sizeof(double) * pp, st));
  pool(&g.counts, sizeof(int64_t) * 4 * (size_t)std::max<int64_t>(p_loc, 1));
}

// Staging blocks are whole groups of 16 SNP rows (layout 2 transposes 16 at a time).
static int64_t staging_rows(int64_t stride, int64_t budget_bytes, int64_t pr) {
  int64_t br = std::max<int64_t>(16, (budget_bytes / stride) & ~int64_t(15));
  return std::min(br, std::max<int64_t>(16, ((pr + 15) / 16) * 16));
}

void GenoOp::build_from_payload(const uint8_t* payload, int64_t p, int64_t nn) {
  if (p <= 0 || nn <= 0) fail(GKB_EINVAL, "genotype operator: empty dimension");
  m = p;
  n = nn;
  starts = partition_rows(p, ctx->nshards_total);
  const int L = (int)ctx->shards.size();
  gs.resize(L);
  const int64_t stride = (nn + 3) / 4;
  for (int i = 0; i < L; ++i) {
    const int64_t r0 = row0(i), pr = rows(i);
    alloc_shard(i, pr, nn);
    Shard& sh = ctx->shards[i];
    ctx->set_device(i);
    const int64_t br = staging_rows(stride, 64ll << 20, pr);
    DevScratch dhold;  // RAII: a throw below must not leak the staging buffers
    PinnedScratch hhold;
    GKB_CUDA(cudaMalloc(&dhold.p, (size_t)(br * stride)));
    GKB_CUDA(cudaMallocHost(&hhold.p, (size_t)(br * stride)));
    uint8_t* dstage = dhold.as<uint8_t>();
    uint8_t* hstage = hhold.as<uint8_t>();
    for (int64_t b0 = 0; b0 < pr; b0 += br) {
      const int64_t rb = std::min(br, pr - b0);
      GKB_CUDA(cudaStreamSynchronize(sh.stream));  // hstage free again
      std::memcpy(hstage, payload + (r0 + b0) * stride, (size_t)(rb * stride));
      GKB_CUDA(cudaMemcpyAsync(dstage, hstage, (size_t)(rb * stride), cudaMemcpyHostToDevice,
                               sh.stream));
      dev::build_lt1(dstage, stride, rb, b0, nn, gs[i].pl1, gs[i].lt1, sh.stream);
      GKB_LAUNCH_CHECK();
      if (!gs[i].single) dev::build_lt2(dstage, stride, rb, b0, nn, gs[i].pl2, gs[i].lt2, sh.stream);
      GKB_LAUNCH_CHECK();
    }
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
  }
  finish_build();
}

// ---------------------------------------------------------------- .bed files
static int64_t count_lines(const char* path) {  // genio.cpp:21-30 (non-empty lines)
  FILE* f = std::fopen(path, "rb");
  if (!f) fail(GKB_EFORMAT, std::string("cannot open ") + path);
  int64_t lines = 0;
  bool nonempty = false;
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, f)) > 0)
    for (size_t i = 0; i < got; ++i) {
      if (buf[i] == '\n') {
        lines += nonempty;
        nonempty = false;
      } else {
        nonempty = true;  // (getline keeps '\r'; a line of just "\r" counts, as there)
      }
    }
  lines += nonempty;  // last line without a newline
  std::fclose(f);
  return lines;
}

void bed_check(const char* bed, const char* bim, const char* fam, int64_t* p, int64_t* n) {
  const int64_t m = count_lines(bim), nn = count_lines(fam);
  FILE* f = std::fopen(bed, "rb");
  if (!f) fail(GKB_EFORMAT, std::string("cannot open ") + bed);
  unsigned char hdr[3] = {0, 0, 0};
  const size_t got = std::fread(hdr, 1, 3, f);
  std::fseek(f, 0, SEEK_END);
  const int64_t size = (int64_t)std::ftell(f);
  std::fclose(f);
  if (got < 3 || size < 3 || hdr[0] != 0x6c || hdr[1] != 0x1b)
    fail(GKB_EFORMAT, std::string(bed) + ": bad magic");
  if (hdr[2] != 0x01)
    fail(GKB_EFORMAT, std::string(bed) + ": only marker-major mode (0x01) is supported");
  const int64_t expected = m * ((nn + 3) / 4) + 3;
  if (size != expected)
    fail(GKB_EFORMAT, std::string(bed) + ": payload size mismatch (expected " +
                          std::to_string(expected) + " bytes, found " + std::to_string(size) + ")");
  *p = m;
  *n = nn;
}

static bool verbose() {
  const char* e = std::getenv("GKB_VERBOSE");
  return e && e[0] == '1';
}
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// positional-read threads per staging block (GKB_READ_THREADS for sweeps)
static unsigned read_threads() {
  static const unsigned t = [] {
    const char* e = std::getenv("GKB_READ_THREADS");
    const int v = e ? std::atoi(e) : 8;  // 16 measured no faster (page-cache copies)
    return (unsigned)std::max(1, std::min(64, v));
  }();
  return t;
}

void GenoOp::build_from_bed_file(const char* bed, int64_t p, int64_t nn) {
  if (p <= 0 || nn <= 0) fail(GKB_EINVAL, "genotype operator: empty dimension");
  const double t0 = now_s();
  double t_alloc = 0.0, t_read = 0.0;
  m = p;
  n = nn;
  starts = partition_rows(p, ctx->nshards_total);
  const int L = (int)ctx->shards.size();
  gs.resize(L);
  const int64_t stride = (nn + 3) / 4;
  const int fd = ::open(bed, O_RDONLY);
  if (fd < 0) fail(GKB_EFORMAT, std::string("cannot open ") + bed);
  try {
    for (int i = 0; i < L; ++i) {
      const int64_t r0 = row0(i), pr = rows(i);
      const double ta = now_s();
      alloc_shard(i, pr, nn);
      Shard& sh = ctx->shards[i];
      ctx->set_device(i);
      // staging block: 16 MB (GKB_STAGE_MB overrides; tests use small blocks to
      // exercise the double buffering); each block is read by several threads
      int64_t budget = 16ll << 20;
      if (const char* e = std::getenv("GKB_STAGE_MB")) budget = std::max<int64_t>(1, atoll(e)) << 20;
      const int64_t br = staging_rows(stride, budget, pr);
      const int nthr = (int)std::max(1u, std::min(read_threads(), std::thread::hardware_concurrency()));
      // scratch held by RAII so a short read or a CUDA error does not leak it
      DevScratch dhold[2];
      EventHolder ehold[2];
      uint8_t* dstage[2] = {nullptr, nullptr};
      uint8_t* hstage[2] = {nullptr, nullptr};
      cudaEvent_t ev[2] = {nullptr, nullptr};
      for (int k = 0; k < 2; ++k) {
        dhold[k].st = sh.stream;
        GKB_CUDA(cudaMallocAsync(&dhold[k].p, (size_t)(br * stride), sh.stream));
        dstage[k] = dhold[k].as<uint8_t>();
        hstage[k] = sh.pinned_stage(k, (size_t)(br * stride));  // cached across loads
        GKB_CUDA(cudaEventCreateWithFlags(&ehold[k].e, cudaEventDisableTiming));
        ev[k] = ehold[k].e;
      }
      t_alloc += now_s() - ta;
      int k = 0;
      for (int64_t b0 = 0; b0 < pr; b0 += br, k ^= 1) {
        const int64_t rb = std::min(br, pr - b0);
        GKB_CUDA(cudaEventSynchronize(ev[k]));  // staging k consumed by its layout builds
        const double tr = now_s();
        // positional reads of this block's records (nthr slices in parallel)
        // while the device works on the other buffer
        const int64_t want = rb * stride;
        const off_t base = (off_t)(3 + (r0 + b0) * stride);
        std::vector<int> bad(nthr, 0);
        auto read_slice = [&](int t) {
          int64_t done = want * t / nthr;
          const int64_t end = want * (t + 1) / nthr;
          while (done < end) {
            const ssize_t r = ::pread(fd, hstage[k] + done, (size_t)(end - done), base + done);
            if (r <= 0) {
              bad[t] = 1;
              return;
            }
            done += r;
          }
        };
        if (nthr == 1 || want < (1 << 20)) {
          read_slice(0);
          for (int t = 1; t < nthr; ++t) read_slice(t);
        } else {
          std::vector<std::thread> pool;
          for (int t = 1; t < nthr; ++t) pool.emplace_back(read_slice, t);
          read_slice(0);
          for (auto& th : pool) th.join();
        }
        for (int t = 0; t < nthr; ++t)
          if (bad[t]) fail(GKB_EFORMAT, std::string(bed) + ": short read");
        t_read += now_s() - tr;
        GKB_CUDA(cudaMemcpyAsync(dstage[k], hstage[k], (size_t)want, cudaMemcpyHostToDevice,
                                 sh.stream));
        dev::build_lt1(dstage[k], stride, rb, b0, nn, gs[i].pl1, gs[i].lt1, sh.stream);
        GKB_LAUNCH_CHECK();
        if (!gs[i].single) dev::build_lt2(dstage[k], stride, rb, b0, nn, gs[i].pl2, gs[i].lt2, sh.stream);
        GKB_LAUNCH_CHECK();
        GKB_CUDA(cudaEventRecord(ev[k], sh.stream));
      }
      GKB_CUDA(cudaStreamSynchronize(sh.stream));  // staging freed / events destroyed by RAII
    }
  } catch (...) {
    ::close(fd);
    throw;
  }
  ::close(fd);
  const double t1 = now_s();
  finish_build();
  if (verbose())
    std::fprintf(stderr, "[gkb] bed ingest: alloc %.4f s, reads %.4f s, stream+build %.4f s, "
                 "finish (counts, lists, scratch) %.4f s\n", t_alloc, t_read,
                 t1 - t0 - t_alloc - t_read, now_s() - t1);
}

void GenoOp::build_from_synth(const dev::SynthDev& sp_in, const gkb_synth_spec* spec) {
  const int64_t p = spec->p, nn = spec->n;
  if (p <= 0 || nn <= 0) fail(GKB_EINVAL, "synth: empty dimension");
  if (spec->npop < 1 || !spec->freq) fail(GKB_EINVAL, "synth: need npop >= 1 and freq");
  if (!spec->pop && !spec->admix) fail(GKB_EINVAL, "synth: need pop or admix");
  m = p;
  n = nn;
  starts = partition_rows(p, ctx->nshards_total);
  const int L = (int)ctx->shards.size();
  gs.resize(L);
  const int64_t stride = (nn + 3) / 4;
  (void)sp_in;
  plan_missing = spec->missing_rate;
  for (int i = 0; i < L; ++i) {
    const int64_t r0 = row0(i), pr = rows(i);
    alloc_shard(i, pr, nn);
    Shard& sh = ctx->shards[i];
    ctx->set_device(i);
    // device copies of the spec arrays
    DevScratch hfreq, hpop, hadmix, hcopy, dhold;  // RAII: freed on a throw too
    double* dfreq = nullptr;
    int32_t* dpop = nullptr;
    double* dadmix = nullptr;
    int32_t* dcopy = nullptr;
    GKB_CUDA(cudaMalloc(&hfreq.p, sizeof(double) * (size_t)(spec->npop * p)));
    dfreq = hfreq.as<double>();
    // stream-ordered copies: a synchronous cudaMemcpy from pageable memory may
    // return before its DMA lands, and the shard stream does not wait for it
    GKB_CUDA(cudaMemcpyAsync(dfreq, spec->freq, sizeof(double) * (size_t)(spec->npop * p),
                             cudaMemcpyHostToDevice, sh.stream));
    if (spec->pop) {
      GKB_CUDA(cudaMalloc(&hpop.p, sizeof(int32_t) * (size_t)nn));
      dpop = hpop.as<int32_t>();
      GKB_CUDA(cudaMemcpyAsync(dpop, spec->pop, sizeof(int32_t) * (size_t)nn,
                               cudaMemcpyHostToDevice, sh.stream));
    } else {
      GKB_CUDA(cudaMalloc(&hadmix.p, sizeof(double) * (size_t)(nn * spec->npop)));
      dadmix = hadmix.as<double>();
      GKB_CUDA(cudaMemcpyAsync(dadmix, spec->admix, sizeof(double) * (size_t)(nn * spec->npop),
                               cudaMemcpyHostToDevice, sh.stream));
    }
    if (spec->copy_from) {
      GKB_CUDA(cudaMalloc(&hcopy.p, sizeof(int32_t) * (size_t)nn));
      dcopy = hcopy.as<int32_t>();
      GKB_CUDA(cudaMemcpyAsync(dcopy, spec->copy_from, sizeof(int32_t) * (size_t)nn,
                               cudaMemcpyHostToDevice, sh.stream));
    }
    dev::SynthDev sd{p, nn, spec->seed, spec->npop, dfreq, dpop, dadmix, spec->missing_rate, dcopy,
                     spec->copy_prob};
    const int64_t br = staging_rows(stride, 256ll << 20, pr);
    GKB_CUDA(cudaMalloc(&dhold.p, (size_t)(br * stride)));
    uint8_t* dstage = dhold.as<uint8_t>();
    for (int64_t b0 = 0; b0 < pr; b0 += br) {
      const int64_t rb = std::min(br, pr - b0);
      dev::synth_bed(sd, r0 + b0, rb, dstage, sh.stream);
      GKB_LAUNCH_CHECK();
      dev::build_lt1(dstage, stride, rb, b0, nn, gs[i].pl1, gs[i].lt1, sh.stream);
      GKB_LAUNCH_CHECK();
      if (!gs[i].single) dev::build_lt2(dstage, stride, rb, b0, nn, gs[i].pl2, gs[i].lt2, sh.stream);
      GKB_LAUNCH_CHECK();
    }
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
  }
  finish_build();
}

// Missing-data handling of a shard: per-CTA lists walked in the epilogue
// (cost grows with the missing count) below the threshold fraction, indicator
// MMAs (flat cost, no list bytes) above it. GKB_MISS_MODE=list|ind forces one.
static bool dense_missing(int64_t nmissing, int64_t p_loc, int64_t n) {
  if (const char* e = std::getenv("GKB_MISS_MODE")) {
    if (std::strcmp(e, "ind") == 0) return true;
    if (std::strcmp(e, "list") == 0) return false;
  }
  double thr = 0.015;
  if (const char* e = std::getenv("GKB_MISS_THRESHOLD")) thr = std::atof(e);
  return (double)nmissing > thr * (double)p_loc * (double)n;
}

void GenoOp::finish_build() {
  const int L = (int)ctx->shards.size();
  counts_host.assign((size_t)(4 * m), 0);
  for (int i = 0; i < L; ++i) {
    GenoShard& g = gs[i];
    Shard& sh = ctx->shards[i];
    ctx->set_device(i);
    dev::marker_counts(g.lt1, g.pl1, g.p_loc, g.n, g.counts, sh.stream);
    GKB_LAUNCH_CHECK();
    if (g.p_loc > 0)
      GKB_CUDA(cudaMemcpyAsync(counts_host.data() + 4 * row0(i), g.counts,
                               sizeof(int64_t) * (size_t)(4 * g.p_loc), cudaMemcpyDeviceToHost,
                               sh.stream));
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
    g.nmissing = 0;
    for (int64_t j = 0; j < g.p_loc; ++j) g.nmissing += counts_host[4 * (row0(i) + j) + 3];
    if (g.p_loc > 0) {  // observed means (orc_marker_means' formula, bit-identical)
      std::vector<double> mh((size_t)g.p_loc);
      for (int64_t j = 0; j < g.p_loc; ++j) {
        const int64_t* c = counts_host.data() + 4 * (row0(i) + j);
        const int64_t obs = c[0] + c[1] + c[2];
        mh[j] = obs > 0 ? (double)(c[1] + 2 * c[2]) / (double)obs : 0.0;
      }
      // (pageable source: staged by the call, the vector may go out of scope)
      GKB_CUDA(cudaMemcpyAsync(g.mean, mh.data(), sizeof(double) * (size_t)g.p_loc,
                               cudaMemcpyHostToDevice, sh.stream));
    }
    g.list_bytes = 0;
    g.ind = g.nmissing > 0 && dense_missing(g.nmissing, g.p_loc, g.n);
    auto pool = [&](auto** ptr, size_t bytes) {
      GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, sh.stream));
    };
    if (g.ind && !g.single) {  // indicator MMAs instead of lists; K2's cm digits
      pool(&g.s2m.dig, sizeof(uint4) * (size_t)(g.pl2.nkc * g.pl2.kt_cta * 64));
      pool(&g.s2m.dexp, sizeof(int) * (size_t)g.pl2.nkc);
      pool(&g.s2m.dsum, sizeof(double) * (size_t)g.pl2.nkc);
    }
    if (g.nmissing > 0 && !g.ind) {
      const int64_t t1 = build_block_lists(g.lt1, g.pl1, sh.stream, &g.m1_off, &g.m1_base,
                                           &g.m1_ent, &g.list_bytes);
      if (t1 != g.nmissing) fail(GKB_ECUDA, "missing-list count mismatch (layout 1)");
    }
    if (g.nmissing > 0 && !g.ind && !g.single) {
      const int64_t t2 = build_block_lists(g.lt2, g.pl2, sh.stream, &g.m2_off, &g.m2_base,
                                           &g.m2_ent, &g.list_bytes);
      if (t2 != g.nmissing) fail(GKB_ECUDA, "missing-list count mismatch (layout 2)");
    }
    if (g.nmissing > 0 && g.single) {  // K2 from layout 1 always walks lists
      const int64_t t2 = build_l1t_lists(g, sh.stream);
      if (t2 != g.nmissing) fail(GKB_ECUDA, "missing-list count mismatch (single layout)");
    }
    alloc_scratch(g.pl1, false, g.s1, sh.stream);
    if (g.single) {  // K2's scratch in the single-layout geometry
      const dev::L1TPlan& lt = g.plt;
      pool(&g.s2.dig, dev::l1t_dig_bytes() * (size_t)lt.nkc);
      pool(&g.s2.dexp, sizeof(int) * (size_t)lt.nkc);
      pool(&g.s2.dsum, sizeof(double) * (size_t)lt.nkc);
      pool(&g.s2.part, sizeof(double) * (size_t)(lt.nkc * lt.rows_pad));
      pool(&g.s2.cm, sizeof(double) * (size_t)(lt.nkc * 1792));
      pool(&g.s2.tick, sizeof(unsigned));
    } else {
      alloc_scratch(g.pl2, true, g.s2, sh.stream);
    }
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
  }
  if (ctx->spmd_mode && ctx->nshards_total > 1) {
    // gather global counts: exact in fp64 (counts < 2^53)
    Shard& s = ctx->shards[0];
    ctx->set_device(0);
    std::vector<double> hc(counts_host.begin(), counts_host.end());
    double* dc = nullptr;
    GKB_CUDA(cudaMalloc(&dc, sizeof(double) * hc.size()));
    // stream-ordered: a synchronous cudaMemcpy from pageable memory may return
    // before its DMA lands, and the allreduce on the shard stream (a
    // non-blocking stream) would read stale counts
    GKB_CUDA(cudaMemcpyAsync(dc, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice,
                             s.stream));
    ctx->allreduce({dc}, (int64_t)hc.size());
    GKB_CUDA(cudaMemcpyAsync(hc.data(), dc, sizeof(double) * hc.size(), cudaMemcpyDeviceToHost,
                             s.stream));
    GKB_CUDA(cudaStreamSynchronize(s.stream));
    cudaFree(dc);
    for (size_t t = 0; t < hc.size(); ++t) counts_host[t] = (int64_t)hc[t];
  }
  alloc_host_api_buffers();
}

void GenoOp::set_scaling(const double* mu, const double* inv_s) {
  const int L = (int)ctx->shards.size();
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    if (rows(i) == 0) continue;
    GKB_CUDA(cudaMemcpyAsync(gs[i].mu, mu + row0(i), sizeof(double) * (size_t)rows(i),
                             cudaMemcpyHostToDevice, ctx->shards[i].stream));
    GKB_CUDA(cudaMemcpyAsync(gs[i].inv_s, inv_s + row0(i), sizeof(double) * (size_t)rows(i),
                             cudaMemcpyHostToDevice, ctx->shards[i].stream));
  }
  ctx->sync_all();
  scaled = true;
}

void GenoOp::get_scaling(double* mu, double* inv_s) {
  const int L = (int)ctx->shards.size();
  std::fill(mu, mu + m, 0.0);
  std::fill(inv_s, inv_s + m, 0.0);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    if (rows(i) == 0) continue;
    GKB_CUDA(cudaMemcpyAsync(mu + row0(i), gs[i].mu, sizeof(double) * (size_t)rows(i),
                             cudaMemcpyDeviceToHost, ctx->shards[i].stream));
    GKB_CUDA(cudaMemcpyAsync(inv_s + row0(i), gs[i].inv_s, sizeof(double) * (size_t)rows(i),
                             cudaMemcpyDeviceToHost, ctx->shards[i].stream));
  }
  ctx->sync_all();
  if (ctx->spmd_mode && ctx->nshards_total > 1) {
    // every rank returns the full vectors: zero-padded rows summed over ranks
    Shard& s = ctx->shards[0];
    ctx->set_device(0);
    DevScratch buf;
    GKB_CUDA(cudaMalloc(&buf.p, sizeof(double) * (size_t)(2 * m)));
    double* d = buf.as<double>();
    GKB_CUDA(cudaMemcpyAsync(d, mu, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, s.stream));
    GKB_CUDA(cudaMemcpyAsync(d + m, inv_s, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice,
                             s.stream));
    ctx->allreduce({d}, 2 * m);
    GKB_CUDA(cudaMemcpyAsync(mu, d, sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost, s.stream));
    GKB_CUDA(cudaMemcpyAsync(inv_s, d + m, sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost,
                             s.stream));
    GKB_CUDA(cudaStreamSynchronize(s.stream));
  }
}

void DevOp::apply_dev_div(const std::vector<const double*>& xraw,
                          const std::vector<const double*>& div,
                          const std::vector<const int*>& gate, const std::vector<double*>& xs,
                          const std::vector<double*>& y) {
  for (size_t i = 0; i < ctx->shards.size(); ++i) {
    ctx->set_device((int)i);
    dev::div_copy_dv(xraw[i], div[i], xs[i], n, ctx->shards[i].stream, gate[i]);
  }
  std::vector<const double*> xc(xs.begin(), xs.end());
  apply_dev(xc, y);
}

void DevOp::adjoint_dev_div(const std::vector<const double*>& yraw,
                            const std::vector<const double*>& div,
                            const std::vector<const int*>& gate, const std::vector<double*>& ys,
                            const std::vector<double*>& z) {
  for (size_t i = 0; i < ctx->shards.size(); ++i) {
    ctx->set_device((int)i);
    dev::div_copy_dv(yraw[i], div[i], ys[i], rows((int)i), ctx->shards[i].stream, gate[i]);
  }
  std::vector<const double*> yc(ys.begin(), ys.end());
  adjoint_dev(yc, z);
}

void GenoOp::apply_dev(const std::vector<const double*>& x, const std::vector<double*>& y) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  for (size_t i = 0; i < gs.size(); ++i) {
    ctx->set_device((int)i);
    dev::k1_apply(gs[i].view(), x[i], y[i], ctx->shards[i].stream, host_out_);
    GKB_LAUNCH_CHECK();
  }
}

// Column pairs through the two-vector kernel (each column bitwise the
// single-vector product); an odd last column goes alone.
// tcgen05 block products (k_pm_blk_tc) for k >= 6 columns, where one pass
// beats ceil(k/2) passes of the two-column kernel;
// GKB_TC_BLOCK=0 disables, =1 uses them from k = 3. Both layouts present;
// lists not required (exact indicator MMAs).
static bool use_tc_block(const GenoShard& g, int64_t k) {
  const char* e = std::getenv("GKB_TC_BLOCK");
  if (e && std::strcmp(e, "0") == 0) return false;
  const int64_t kmin = (e && std::strcmp(e, "1") == 0) ? 3 : 6;
  return k >= kmin && !g.single;
}

static void ensure_tc(dev::TcScratch& t, const dev::PMPlan& pl, int kmax, bool k2,
                      cudaStream_t st) {
  if (t.kmax >= kmax) return;
  void* ptrs[] = {t.dig, t.dig2, t.dexp, t.dexp2, t.dsum, t.part};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, st);
  t = dev::TcScratch{};
  auto pool = [&](auto** ptr, size_t bytes) {
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, st));
  };
  pool(&t.dig, dev::tc_dig_bytes(pl, kmax));
  if (k2) pool(&t.dig2, dev::tc_dig_bytes(pl, kmax));
  const int64_t nkc = dev::tc_nkc(pl);
  pool(&t.dexp, sizeof(int) * (size_t)(kmax * nkc));
  if (k2) pool(&t.dexp2, sizeof(int) * (size_t)(kmax * nkc));
  pool(&t.dsum, sizeof(double) * (size_t)(kmax * nkc));
  pool(&t.part, sizeof(double) * (size_t)kmax * (size_t)nkc * (size_t)pl.rows_pad);
  t.kmax = kmax;
}

void GenoOp::apply_block_dev(const std::vector<const double*>& X, int64_t ldx, int64_t k,
                             const std::vector<double*>& Y, const std::vector<int64_t>& ldy) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  if (use_tc_block(gs[0], k)) {
    for (int64_t c0 = 0; c0 < k; c0 += 16) {
      const int kk = (int)std::min<int64_t>(16, k - c0);
      for (size_t i = 0; i < gs.size(); ++i) {
        ctx->set_device((int)i);
        GenoShard& g = gs[i];
        cudaStream_t st = ctx->shards[i].stream;
        ensure_tc(g.tc1, g.pl1, std::max(kk, (int)std::min<int64_t>(k, 16)), false, st);
        dev::k1_apply_tc(g.view(), g.tc1, X[i] + c0 * ldx, ldx, kk, Y[i] + c0 * ldy[i], ldy[i],
                         st);
        GKB_LAUNCH_CHECK();
      }
    }
    return;
  }
  int64_t c = 0;
  for (; c + 2 <= k; c += 2)
    for (size_t i = 0; i < gs.size(); ++i) {
      ctx->set_device((int)i);
      GenoShard& g = gs[i];
      cudaStream_t st = ctx->shards[i].stream;
      if (!g.s1b.part && !g.ind) alloc_scratch(g.pl1, false, g.s1b, st);
      dev::k1_apply2(g.view(), g.s1b, X[i] + c * ldx, X[i] + (c + 1) * ldx, Y[i] + c * ldy[i],
                     Y[i] + (c + 1) * ldy[i], st);
      GKB_LAUNCH_CHECK();
    }
  if (c < k) {
    const int L = (int)gs.size();
    std::vector<const double*> xi(L);
    std::vector<double*> yi(L);
    for (int i = 0; i < L; ++i) {
      xi[i] = X[i] + c * ldx;
      yi[i] = Y[i] + c * ldy[i];
    }
    apply_dev(xi, yi);
  }
}

void GenoOp::adjoint_block_dev(const std::vector<const double*>& Yb,
                               const std::vector<int64_t>& ldyb, int64_t k,
                               const std::vector<double*>& Z, int64_t ldz) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  const int L = (int)gs.size();
  if (use_tc_block(gs[0], k)) {
    for (int64_t c0 = 0; c0 < k; c0 += 16) {
      const int kk = (int)std::min<int64_t>(16, k - c0);
      for (int i = 0; i < L; ++i) {
        ctx->set_device(i);
        GenoShard& g = gs[i];
        cudaStream_t st = ctx->shards[i].stream;
        ensure_tc(g.tc2, g.pl2, std::max(kk, (int)std::min<int64_t>(k, 16)), true, st);
        dev::k2_adjoint_tc(g.view(), g.tc2, Yb[i] + c0 * ldyb[i], ldyb[i], kk, Z[i] + c0 * ldz,
                           ldz, st);
        GKB_LAUNCH_CHECK();
      }
      for (int64_t q = c0; q < c0 + kk; ++q) {  // cross-shard sums, column by column
        std::vector<double*> zq(L);
        for (int i = 0; i < L; ++i) zq[i] = Z[i] + q * ldz;
        ctx->allreduce(zq, n);
      }
    }
    return;
  }
  int64_t c = 0;
  for (; c + 2 <= k; c += 2) {
    for (int i = 0; i < L; ++i) {
      ctx->set_device(i);
      GenoShard& g = gs[i];
      cudaStream_t st = ctx->shards[i].stream;
      if (!g.s2b.part && !g.ind && !g.single) alloc_scratch(g.pl2, true, g.s2b, st);
      dev::k2_adjoint2(g.view(), g.s2b, Yb[i] + c * ldyb[i], Yb[i] + (c + 1) * ldyb[i],
                       Z[i] + c * ldz, Z[i] + (c + 1) * ldz, st);
      GKB_LAUNCH_CHECK();
    }
    for (int64_t q = c; q < c + 2; ++q) {  // cross-shard sums, column by column
      std::vector<double*> zq(L);
      for (int i = 0; i < L; ++i) zq[i] = Z[i] + q * ldz;
      ctx->allreduce(zq, n);
    }
  }
  if (c < k) {
    std::vector<const double*> yi(L);
    std::vector<double*> zi(L);
    for (int i = 0; i < L; ++i) {
      yi[i] = Yb[i] + c * ldyb[i];
      zi[i] = Z[i] + c * ldz;
    }
    adjoint_dev(yi, zi);
  }
}

void GenoOp::apply_dev_div(const std::vector<const double*>& xraw,
                           const std::vector<const double*>& div,
                           const std::vector<const int*>& gate, const std::vector<double*>& xs,
                           const std::vector<double*>& y) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  for (size_t i = 0; i < gs.size(); ++i) {
    ctx->set_device((int)i);
    dev::DivIn di;
    di.div = div[i];
    di.store = xs[i];
    di.gate = gate[i];
    dev::k1_apply(gs[i].view(), xraw[i], y[i], ctx->shards[i].stream, host_out_, di);
    GKB_LAUNCH_CHECK();
  }
}

void GenoOp::adjoint_dev_div(const std::vector<const double*>& yraw,
                             const std::vector<const double*>& div,
                             const std::vector<const int*>& gate, const std::vector<double*>& ys,
                             const std::vector<double*>& z) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  for (size_t i = 0; i < gs.size(); ++i) {
    ctx->set_device((int)i);
    dev::DivIn di;
    di.div = div[i];
    di.store = ys[i];
    di.gate = gate[i];
    dev::k2_adjoint(gs[i].view(), yraw[i], z[i], ctx->shards[i].stream, di);
    GKB_LAUNCH_CHECK();
  }
  ctx->allreduce(z, n);
}

void GenoOp::adjoint_dev(const std::vector<const double*>& y, const std::vector<double*>& z) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  for (size_t i = 0; i < gs.size(); ++i) {
    ctx->set_device((int)i);
    dev::k2_adjoint(gs[i].view(), y[i], z[i], ctx->shards[i].stream);
    GKB_LAUNCH_CHECK();
  }
  ctx->allreduce(z, n);
}

// Per-marker scan: [y, 1, Z] block product on the device (two columns per
// pass), the (k+1) x (k+1) nuisance algebra on the host, one thread per marker.
void GenoOp::marker_scan(const double* y, const double* Z, int64_t k, bool unbiased,
                         double* beta, double* se, double* icpt, double* sig2, int32_t* dep) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  if (ctx->spmd_mode && ctx->nshards_total > 1)
    fail(GKB_ELOGIC, "marker_scan: SPMD operators use the host scan");
  const int K = (int)(k + 1);
  const int64_t nn = n;
  // C = [1, Z]; A = C'C, w = C'y, A^-1 (Gauss-Jordan with partial pivoting)
  std::vector<double> A((size_t)(K * K), 0.0), wv((size_t)K, 0.0), X((size_t)(nn * (K + 1)));
  auto Cv = [&](int64_t s2, int a) { return a == 0 ? 1.0 : Z[(int64_t)(a - 1) * nn + s2]; };
  for (int64_t s2 = 0; s2 < nn; ++s2) {
    X[s2] = y[s2];
    for (int a = 0; a < K; ++a) {
      const double ca = Cv(s2, a);
      X[(int64_t)(1 + a) * nn + s2] = ca;
      wv[a] += ca * y[s2];
      for (int b = 0; b <= a; ++b) A[a + b * K] += ca * Cv(s2, b);
    }
  }
  for (int a = 0; a < K; ++a)
    for (int b = a + 1; b < K; ++b) A[a + b * K] = A[b + a * K];
  std::vector<double> Ai((size_t)(K * K), 0.0), M(A);
  for (int a = 0; a < K; ++a) Ai[a + a * K] = 1.0;
  for (int c = 0; c < K; ++c) {
    int piv = c;
    for (int r2 = c + 1; r2 < K; ++r2)
      if (std::fabs(M[r2 + c * K]) > std::fabs(M[piv + c * K])) piv = r2;
    if (M[piv + c * K] == 0.0) fail(GKB_ELOGIC, "marker_scan: nuisance design is singular");
    for (int j = 0; j < K; ++j) {
      std::swap(M[c + j * K], M[piv + j * K]);
      std::swap(Ai[c + j * K], Ai[piv + j * K]);
    }
    const double dv = M[c + c * K];
    for (int j = 0; j < K; ++j) {
      M[c + j * K] /= dv;
      Ai[c + j * K] /= dv;
    }
    for (int r2 = 0; r2 < K; ++r2)
      if (r2 != c) {
        const double f = M[r2 + c * K];
        if (f == 0.0) continue;
        for (int j = 0; j < K; ++j) {
          M[r2 + j * K] -= f * M[c + j * K];
          Ai[r2 + j * K] -= f * Ai[c + j * K];
        }
      }
  }
  double yy = 0.0;
  for (int64_t s2 = 0; s2 < nn; ++s2) yy += y[s2] * y[s2];
  double wAw = 0.0, a0w = 0.0;
  for (int a = 0; a < K; ++a)
    for (int b = 0; b < K; ++b) {
      wAw += wv[a] * Ai[a + b * K] * wv[b];
      if (a == 0) a0w += Ai[0 + b * K] * wv[b];
    }
  const double yyc = yy - wAw;
  const double denom = unbiased ? (double)(nn - (K + 1)) : (double)nn;
  const int L = (int)gs.size();
  int64_t rmax = 1;
  for (int i = 0; i < L; ++i) rmax = std::max(rmax, rows(i));
  ensure_block_buffers(nn * (K + 1), rmax * (K + 1) + 5 * rmax + 2 * (K * K + K));
  std::vector<const double*> xb(L);
  std::vector<double*> yb(L);
  std::vector<int64_t> ld(L);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    GKB_CUDA(cudaMemcpyAsync(bin_[i], X.data(), sizeof(double) * (size_t)(nn * (K + 1)),
                             cudaMemcpyHostToDevice, ctx->shards[i].stream));
    xb[i] = bin_[i];
    yb[i] = bout_[i];
    ld[i] = rows(i);
  }
  apply_block_dev(xb, nn, K + 1, yb, ld);
  std::vector<double> aw(Ai);
  aw.insert(aw.end(), wv.begin(), wv.end());
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    cudaStream_t st = ctx->shards[i].stream;
    const int64_t r = rows(i);
    double* base = bout_[i] + r * (K + 1);
    double* dAi = base + 5 * rmax;
    GKB_CUDA(cudaMemcpyAsync(dAi, aw.data(), sizeof(double) * aw.size(), cudaMemcpyHostToDevice, st));
    int* ddep = reinterpret_cast<int*>(base + 4 * rmax);
    dev::marker_scan(gs[i].view(), bout_[i], std::max<int64_t>(r, 1), K, dAi, dAi + K * K, yyc,
                     a0w, denom, gs[i].counts, base, base + rmax, base + 2 * rmax, base + 3 * rmax,
                     ddep, st);
    GKB_LAUNCH_CHECK();
    const int64_t r0 = row0(i);
    Shard& sh = ctx->shards[i];
    GKB_CUDA(cudaStreamSynchronize(st));
    d2h_staged(sh, beta + r0, base, sizeof(double) * (size_t)r);
    d2h_staged(sh, se + r0, base + rmax, sizeof(double) * (size_t)r);
    d2h_staged(sh, icpt + r0, base + 2 * rmax, sizeof(double) * (size_t)r);
    d2h_staged(sh, sig2 + r0, base + 3 * rmax, sizeof(double) * (size_t)r);
    d2h_staged(sh, dep + r0, ddep, sizeof(int32_t) * (size_t)r);
  }
  mvps += K + 1;
}

int64_t GenoOp::packed_bytes() const {
  int64_t b = 0;
  const int64_t stride = (n + 3) / 4;
  for (const auto& g : gs) b += g.p_loc * stride;
  return b;
}

int64_t GenoOp::device_bytes() const {
  int64_t b = 0;
  for (const auto& g : gs) {
    b += 4 * (dev::pm_words(g.pl1) + (g.single ? 0 : dev::pm_words(g.pl2)));
    b += g.list_bytes + 16 * g.pl1.rows_pad;  // missing lists, mu + inv_s
  }
  return b;
}

void GenoOp::read_bed(int64_t r0, int64_t nrows, uint8_t* out) {
  if (r0 < 0 || nrows < 0 || r0 + nrows > m) fail(GKB_EINVAL, "read_bed: row range out of bounds");
  const int64_t stride = (n + 3) / 4;
  const int L = (int)ctx->shards.size();
  for (int i = 0; i < L; ++i) {
    const int64_t a = std::max(r0, row0(i)), b = std::min(r0 + nrows, row0(i) + rows(i));
    if (a >= b) continue;
    ctx->set_device(i);
    uint8_t* d = nullptr;
    GKB_CUDA(cudaMalloc(&d, (size_t)((b - a) * stride)));
    dev::layout_to_bed(gs[i].lt1, gs[i].pl1, n, a - row0(i), b - a, d, ctx->shards[i].stream);
    GKB_LAUNCH_CHECK();
    GKB_CUDA(cudaMemcpyAsync(out + (a - r0) * stride, d, (size_t)((b - a) * stride),
                             cudaMemcpyDeviceToHost, ctx->shards[i].stream));
    GKB_CUDA(cudaStreamSynchronize(ctx->shards[i].stream));
    cudaFree(d);
  }
}

// ---------------------------------------------------------------- DenseOp
DenseOp::~DenseOp() {
  for (size_t i = 0; i < X.size(); ++i) {
    cudaSetDevice(ctx->shards[i].dev);
    if (X[i]) cudaFree(X[i]);
  }
}

void DenseOp::build(const double* Xh, int64_t mm, int64_t nn) {
  if (mm <= 0 || nn <= 0) fail(GKB_EINVAL, "dense operator: empty dimension");
  m = mm;
  n = nn;
  starts = partition_rows(mm, ctx->nshards_total);
  const int L = (int)ctx->shards.size();
  X.assign(L, nullptr);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    const int64_t r = rows(i);
    GKB_CUDA(cudaMalloc(&X[i], sizeof(double) * (size_t)std::max<int64_t>(r * nn, 1)));
    if (r > 0)
      GKB_CUDA(cudaMemcpy2D(X[i], sizeof(double) * (size_t)r, Xh + row0(i), sizeof(double) * (size_t)mm,
                            sizeof(double) * (size_t)r, (size_t)nn, cudaMemcpyHostToDevice));
    ctx->shards[i].ensure_partial(dev::red_blocks(r) * (nn + 1) + 16);
  }
  alloc_host_api_buffers();
}

void DenseOp::apply_dev(const std::vector<const double*>& x, const std::vector<double*>& y) {
  for (size_t i = 0; i < X.size(); ++i) {
    ctx->set_device((int)i);
    Shard& s = ctx->shards[i];
    const int64_t r = rows((int)i);
    if (r == 0) continue;
    dev::gemv_n(X[i], r, r, n, x[i], y[i], 0.0, 1.0, false, s.rs, nullptr, s.stream);
    GKB_LAUNCH_CHECK();
  }
}

void DenseOp::adjoint_dev(const std::vector<const double*>& y, const std::vector<double*>& z) {
  for (size_t i = 0; i < X.size(); ++i) {
    ctx->set_device((int)i);
    Shard& s = ctx->shards[i];
    const int64_t r = rows((int)i);
    dev::gemv_t(X[i], std::max<int64_t>(r, 1), r, n, y[i], false, s.rs, z[i], s.stream);
    GKB_LAUNCH_CHECK();
  }
  ctx->allreduce(z, n);
}

}  // namespace gkb
