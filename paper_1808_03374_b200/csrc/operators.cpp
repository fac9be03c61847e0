// Device operators: the packed genotype operator (replacing the reference's
// DenseOperator over the imputed, standardized matrix) and a device
// DenseOperator (linop.hpp:43-64). Rows (reference markers) are sharded;
// columns (samples) are replicated.
#include <algorithm>
#include <cmath>
#include <cstring>

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
    if (ctx->use_nccl && ctx->nshards_total > 1)
      GKB_CUDA(cudaMalloc(&yfull[i], sizeof(double) * (size_t)std::max<int64_t>(m, 1)));
  }
}

void DevOp::apply_host(const double* x, double* y) {
  const int L = (int)ctx->shards.size();
  std::vector<const double*> xi(L);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    GKB_CUDA(cudaMemcpyAsync(xbuf[i], x, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice,
                             ctx->shards[i].stream));
    xi[i] = xbuf[i];
  }
  apply_dev(xi, ybuf);
  if (ctx->use_nccl && ctx->nshards_total > 1) {
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
// Per-CTA missing lists of one plan: count pass, per-block scan on device,
// block bases scanned on the host (nblk values), fill pass. Returns the number
// of entries (== the shard's missing count).
template <class Launch>
static int64_t build_block_lists(int64_t nblk, int span, cudaStream_t st, uint32_t** off,
                                 int64_t** base, uint16_t** ent, int64_t* bytes, Launch launch) {
  uint32_t* cnt = nullptr;
  int64_t* tot = nullptr;
  GKB_CUDA(cudaMalloc(&cnt, sizeof(uint32_t) * (size_t)(nblk * span)));
  GKB_CUDA(cudaMalloc(&tot, sizeof(int64_t) * (size_t)nblk));
  GKB_CUDA(cudaMalloc(off, sizeof(uint32_t) * (size_t)(nblk * (span + 1))));
  launch(false, cnt, nullptr, nullptr, nullptr);
  GKB_LAUNCH_CHECK();
  dev::block_scan(cnt, nblk, span, *off, tot, st);
  GKB_LAUNCH_CHECK();
  std::vector<int64_t> h((size_t)nblk);
  GKB_CUDA(cudaMemcpyAsync(h.data(), tot, sizeof(int64_t) * (size_t)nblk, cudaMemcpyDeviceToHost, st));
  GKB_CUDA(cudaStreamSynchronize(st));
  cudaFree(cnt);
  cudaFree(tot);
  int64_t total = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t c = h[b];
    h[b] = total;
    total += c;
  }
  GKB_CUDA(cudaMalloc(base, sizeof(int64_t) * (size_t)nblk));
  GKB_CUDA(cudaMemcpy(*base, h.data(), sizeof(int64_t) * (size_t)nblk, cudaMemcpyHostToDevice));
  GKB_CUDA(cudaMalloc(ent, sizeof(uint16_t) * (size_t)std::max<int64_t>(total, 1)));
  launch(true, nullptr, *off, *base, *ent);
  GKB_LAUNCH_CHECK();
  *bytes += (int64_t)(sizeof(uint32_t) * nblk * (span + 1) + sizeof(int64_t) * nblk +
                      sizeof(uint16_t) * total);
  return total;
}

dev::GenoView GenoShard::view() const {
  dev::GenoView v;
  v.layA = layA;
  v.layB = layB;
  v.p_loc = p_loc;
  v.n = n;
  v.W = W;
  v.P4 = P4;
  v.mu = mu;
  v.inv_s = inv_s;
  const bool lists = nmissing > 0;
  v.m1_off = lists ? m1_off : nullptr;
  v.m1_base = m1_base;
  v.m1_ent = m1_ent;
  v.m2_off = lists ? m2_off : nullptr;
  v.m2_base = m2_base;
  v.m2_ent = m2_ent;
  v.nmissing = nmissing;
  return v;
}

GenoOp::~GenoOp() {
  for (size_t i = 0; i < gs.size(); ++i) {
    cudaSetDevice(ctx->shards[i].dev);
    GenoShard& g = gs[i];
    void* ptrs[] = {g.layA,   g.layB,   g.mu,    g.inv_s,  g.counts, g.m1_off, g.m1_base,
                    g.m1_ent, g.m2_off, g.m2_base, g.m2_ent, g.ypart, g.zpart};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
}

void GenoOp::alloc_shard(int i, int64_t p_loc, int64_t nn) {
  GenoShard& g = gs[i];
  g.p_loc = p_loc;
  g.n = nn;
  g.W = (nn + 15) / 16;
  g.P4 = (p_loc + 3) / 4;
  ctx->set_device(i);
  const size_t chunks = (size_t)std::max<int64_t>(g.P4 * g.W, 1);
  GKB_CUDA(cudaMalloc(&g.layA, sizeof(uint4) * chunks));
  GKB_CUDA(cudaMalloc(&g.layB, sizeof(uint4) * chunks));
  GKB_CUDA(cudaMemsetAsync(g.layA, 0, sizeof(uint4) * chunks, ctx->shards[i].stream));
  GKB_CUDA(cudaMemsetAsync(g.layB, 0, sizeof(uint4) * chunks, ctx->shards[i].stream));
  const size_t pp = (size_t)std::max<int64_t>(4 * g.P4, 4);
  GKB_CUDA(cudaMalloc(&g.mu, sizeof(double) * pp));
  GKB_CUDA(cudaMalloc(&g.inv_s, sizeof(double) * pp));
  GKB_CUDA(cudaMemsetAsync(g.mu, 0, sizeof(double) * pp, ctx->shards[i].stream));
  GKB_CUDA(cudaMemsetAsync(g.inv_s, 0, sizeof(double) * pp, ctx->shards[i].stream));
  GKB_CUDA(cudaMalloc(&g.counts, sizeof(int64_t) * 4 * pp));  // [n0,n1,n2,nmiss] per row
}

void GenoOp::build_from_payload(const uint8_t* payload, int64_t p, int64_t nn) {
  if (p <= 0 || nn <= 0) fail(GKB_EINVAL, "genotype operator: empty dimension");
  m = p;
  n = nn;
  starts = partition_rows(p, ctx->nshards_total);
  const int L = (int)ctx->shards.size();
  gs.resize(L);
  const int64_t stride = (nn + 3) / 4;
  const int64_t max_block_bytes = 64ll << 20;
  int64_t block_rows = std::max<int64_t>(4, (max_block_bytes / stride) & ~int64_t(3));
  for (int i = 0; i < L; ++i) {
    const int64_t r0 = row0(i), pr = rows(i);
    alloc_shard(i, pr, nn);
    Shard& sh = ctx->shards[i];
    ctx->set_device(i);
    const int64_t br = std::min(block_rows, std::max<int64_t>(4, ((pr + 3) / 4) * 4));
    uint8_t* dstage = nullptr;
    uint8_t* hstage = nullptr;
    GKB_CUDA(cudaMalloc(&dstage, (size_t)(br * stride)));
    GKB_CUDA(cudaMallocHost(&hstage, (size_t)(br * stride)));
    for (int64_t b0 = 0; b0 < pr; b0 += br) {
      const int64_t rb = std::min(br, pr - b0);
      GKB_CUDA(cudaStreamSynchronize(sh.stream));  // hstage free again
      std::memcpy(hstage, payload + (r0 + b0) * stride, (size_t)(rb * stride));
      GKB_CUDA(cudaMemcpyAsync(dstage, hstage, (size_t)(rb * stride), cudaMemcpyHostToDevice,
                               sh.stream));
      dev::build_layouts(dstage, stride, rb, b0 / 4, nn, gs[i].W, gs[i].P4, gs[i].layA, gs[i].layB,
                         sh.stream);
      GKB_LAUNCH_CHECK();
    }
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
    cudaFree(dstage);
    cudaFreeHost(hstage);
  }
  finish_build();
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
  const int64_t block_rows = std::max<int64_t>(4, ((256ll << 20) / stride) & ~int64_t(3));
  (void)sp_in;
  for (int i = 0; i < L; ++i) {
    const int64_t r0 = row0(i), pr = rows(i);
    alloc_shard(i, pr, nn);
    Shard& sh = ctx->shards[i];
    ctx->set_device(i);
    // device copies of the spec arrays
    double* dfreq = nullptr;
    int32_t* dpop = nullptr;
    double* dadmix = nullptr;
    int32_t* dcopy = nullptr;
    GKB_CUDA(cudaMalloc(&dfreq, sizeof(double) * (size_t)(spec->npop * p)));
    GKB_CUDA(cudaMemcpy(dfreq, spec->freq, sizeof(double) * (size_t)(spec->npop * p),
                        cudaMemcpyHostToDevice));
    if (spec->pop) {
      GKB_CUDA(cudaMalloc(&dpop, sizeof(int32_t) * (size_t)nn));
      GKB_CUDA(cudaMemcpy(dpop, spec->pop, sizeof(int32_t) * (size_t)nn, cudaMemcpyHostToDevice));
    } else {
      GKB_CUDA(cudaMalloc(&dadmix, sizeof(double) * (size_t)(nn * spec->npop)));
      GKB_CUDA(cudaMemcpy(dadmix, spec->admix, sizeof(double) * (size_t)(nn * spec->npop),
                          cudaMemcpyHostToDevice));
    }
    if (spec->copy_from) {
      GKB_CUDA(cudaMalloc(&dcopy, sizeof(int32_t) * (size_t)nn));
      GKB_CUDA(cudaMemcpy(dcopy, spec->copy_from, sizeof(int32_t) * (size_t)nn,
                          cudaMemcpyHostToDevice));
    }
    dev::SynthDev sd{p, nn, spec->seed, spec->npop, dfreq, dpop, dadmix, spec->missing_rate, dcopy,
                     spec->copy_prob};
    const int64_t br = std::min(block_rows, std::max<int64_t>(4, ((pr + 3) / 4) * 4));
    uint8_t* dstage = nullptr;
    GKB_CUDA(cudaMalloc(&dstage, (size_t)(br * stride)));
    for (int64_t b0 = 0; b0 < pr; b0 += br) {
      const int64_t rb = std::min(br, pr - b0);
      dev::synth_bed(sd, r0 + b0, rb, dstage, sh.stream);
      GKB_LAUNCH_CHECK();
      dev::build_layouts(dstage, stride, rb, b0 / 4, nn, gs[i].W, gs[i].P4, gs[i].layA, gs[i].layB,
                         sh.stream);
      GKB_LAUNCH_CHECK();
    }
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
    cudaFree(dstage);
    cudaFree(dfreq);
    if (dpop) cudaFree(dpop);
    if (dadmix) cudaFree(dadmix);
    if (dcopy) cudaFree(dcopy);
  }
  finish_build();
}

void GenoOp::finish_build() {
  const int L = (int)ctx->shards.size();
  counts_host.assign((size_t)(4 * m), 0);
  for (int i = 0; i < L; ++i) {
    GenoShard& g = gs[i];
    Shard& sh = ctx->shards[i];
    ctx->set_device(i);
    dev::marker_counts(g.layA, g.P4, g.W, g.p_loc, g.n, g.counts, sh.stream);
    GKB_LAUNCH_CHECK();
    if (g.p_loc > 0)
      GKB_CUDA(cudaMemcpyAsync(counts_host.data() + 4 * row0(i), g.counts,
                               sizeof(int64_t) * (size_t)(4 * g.p_loc), cudaMemcpyDeviceToHost,
                               sh.stream));
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
    g.nmissing = 0;
    for (int64_t j = 0; j < g.p_loc; ++j) g.nmissing += counts_host[4 * (row0(i) + j) + 3];
    g.k1 = dev::k1_plan(g.W, g.P4);
    g.k2 = dev::k2_plan(g.W, g.P4);
    g.list_bytes = 0;
    if (g.nmissing > 0) {
      const uint4* A = g.layA;
      const int64_t P4 = g.P4, W = g.W;
      const dev::K1Plan k1 = g.k1;
      const dev::K2Plan k2 = g.k2;
      const int64_t t1 = build_block_lists(
          k1.grid_x * k1.ntiles, 128, sh.stream, &g.m1_off, &g.m1_base, &g.m1_ent, &g.list_bytes,
          [&](bool fill, uint32_t* cnt, const uint32_t* off, const int64_t* base, uint16_t* ent) {
            dev::miss_lists_k1(A, P4, W, k1, fill, cnt, off, base, ent, sh.stream);
          });
      const int64_t t2 = build_block_lists(
          k2.grid_x * k2.nchunks, 512, sh.stream, &g.m2_off, &g.m2_base, &g.m2_ent, &g.list_bytes,
          [&](bool fill, uint32_t* cnt, const uint32_t* off, const int64_t* base, uint16_t* ent) {
            dev::miss_lists_k2(A, P4, W, k2, fill, cnt, off, base, ent, sh.stream);
          });
      if (t1 != g.nmissing || t2 != g.nmissing) fail(GKB_ECUDA, "missing-list count mismatch");
    }
    GKB_CUDA(cudaMalloc(&g.ypart, sizeof(double) * (size_t)std::max<int64_t>(
                                      (int64_t)g.k1.ntiles * 4 * g.P4, 1)));
    GKB_CUDA(cudaMalloc(&g.zpart, sizeof(double) * (size_t)std::max<int64_t>(
                                      (int64_t)g.k2.nchunks * 16 * g.W, 1)));
    if (g.k1.smem > 48 * 1024)
      fail(GKB_EINVAL, "K1 tile exceeds 48 KB of shared memory");
    GKB_CUDA(cudaStreamSynchronize(sh.stream));
  }
  if (ctx->use_nccl && ctx->nshards_total > 1) {
    // gather global counts: exact in fp64 (counts < 2^53)
    Shard& s = ctx->shards[0];
    ctx->set_device(0);
    std::vector<double> hc(counts_host.begin(), counts_host.end());
    double* dc = nullptr;
    GKB_CUDA(cudaMalloc(&dc, sizeof(double) * hc.size()));
    GKB_CUDA(cudaMemcpy(dc, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice));
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
}

void GenoOp::apply_dev(const std::vector<const double*>& x, const std::vector<double*>& y) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  for (size_t i = 0; i < gs.size(); ++i) {
    ctx->set_device((int)i);
    dev::k1_apply(gs[i].view(), gs[i].k1, x[i], gs[i].ypart, y[i], ctx->shards[i].stream);
    GKB_LAUNCH_CHECK();
  }
}

void GenoOp::adjoint_dev(const std::vector<const double*>& y, const std::vector<double*>& z) {
  if (!scaled) fail(GKB_ELOGIC, "genotype operator: scaling not set (call standardize)");
  for (size_t i = 0; i < gs.size(); ++i) {
    ctx->set_device((int)i);
    dev::k2_adjoint(gs[i].view(), gs[i].k2, y[i], gs[i].zpart, z[i], ctx->shards[i].stream);
    GKB_LAUNCH_CHECK();
  }
  ctx->allreduce(z, n);
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
    b += 2 * 16 * g.P4 * g.W;
    b += g.list_bytes + 16 * 4 * g.P4;  // missing lists, mu + inv_s
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
    dev::layout_to_bed(gs[i].layA, gs[i].P4, gs[i].W, n, a - row0(i), b - a, d,
                       ctx->shards[i].stream);
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
