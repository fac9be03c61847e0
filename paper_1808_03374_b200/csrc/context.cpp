// Context: shards, streams, communicator (local fixed-order device sums or
// NCCL allreduce over NVLink), and the row partition used for SNP sharding.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <thread>
#include <vector>
#include "host.hpp"

namespace gkb {

namespace {
void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(GKB_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

void Shard::ensure_partial(int64_t doubles) {
  if (rs.cap >= doubles) return;
  GKB_CUDA(cudaSetDevice(dev));
  if (rs.partial) GKB_CUDA(cudaFree(rs.partial));
  const int64_t cap = std::max<int64_t>(doubles, 1 << 16);
  GKB_CUDA(cudaMalloc(&rs.partial, sizeof(double) * (size_t)cap));
  rs.cap = cap;
}

void Shard::ensure_res(int64_t doubles) {
  if (res_cap >= doubles) return;
  GKB_CUDA(cudaSetDevice(dev));
  if (stream) GKB_CUDA(cudaStreamSynchronize(stream));
  const int64_t cap = std::max<int64_t>(doubles, kResCap);
  double* d = nullptr;
  double* h = nullptr;
  GKB_CUDA(cudaMalloc(&d, sizeof(double) * (size_t)cap));
  if (cudaMallocHost(&h, sizeof(double) * (size_t)cap) != cudaSuccess) {
    cudaFree(d);
    fail(GKB_EOOM, "ensure_res: cudaMallocHost failed");
  }
  if (dres) cudaFree(dres);
  if (hres) cudaFreeHost(hres);
  dres = d;
  hres = h;
  res_cap = cap;
}

uint8_t* Shard::pinned_stage(int k, size_t bytes) {
  if (bytes > hstage_bytes) {
    for (int q = 0; q < 2; ++q) {
      if (hstage[q]) cudaFreeHost(hstage[q]);
      hstage[q] = nullptr;
    }
    for (int q = 0; q < 2; ++q) GKB_CUDA(cudaMallocHost(&hstage[q], bytes));
    hstage_bytes = bytes;
  }
  return hstage[k];
}

// Device -> pageable host memory through the shard's page-locked staging:
// chunks of <= 8 MB double-buffered (the next chunk's DMA runs while the
// previous one is copied out), each chunk's host copy split over threads.
// A direct copy into fresh pageable memory runs at ~2 GB/s (page faults plus
// the driver's own staging). Synchronous.
void d2h_staged(Shard& s, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  const size_t chunk = std::min<size_t>(bytes, (size_t)8 << 20);
  uint8_t* stage[2] = {s.pinned_stage(0, chunk), s.pinned_stage(1, chunk)};
  cudaEvent_t ev[2];
  for (auto& e : ev) GKB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const size_t nchunks = (bytes + chunk - 1) / chunk;
  auto issue = [&](size_t c) {
    const size_t off = c * chunk, len = std::min(chunk, bytes - off);
    GKB_CUDA(cudaMemcpyAsync(stage[c & 1], static_cast<const uint8_t*>(src) + off, len,
                             cudaMemcpyDeviceToHost, s.stream));
    GKB_CUDA(cudaEventRecord(ev[c & 1], s.stream));
  };
  issue(0);
  for (size_t c = 0; c < nchunks; ++c) {
    GKB_CUDA(cudaEventSynchronize(ev[c & 1]));
    if (c + 1 < nchunks) issue(c + 1);
    const size_t off = c * chunk, len = std::min(chunk, bytes - off);
    const int T = len >= ((size_t)1 << 20) ? 8 : 1;
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
      const size_t a = len * t / T, b = len * (t + 1) / T;
      auto job = [=] { std::memcpy(static_cast<uint8_t*>(dst) + off + a, stage[c & 1] + a, b - a); };
      if (t + 1 < T) th.emplace_back(job); else job();
    }
    for (auto& x : th) x.join();
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

static void init_shard(Shard& s, int index, int dev) {
  s.index = index;
  s.dev = dev;
  GKB_CUDA(cudaSetDevice(dev));
  GKB_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  // stream-ordered allocations (layouts, staging) come from the device's
  // default pool; keep freed memory in the pool so rebuilding an operator of
  // the same size does not go back to the driver
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  s.ensure_res(kResCap);
  GKB_CUDA(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
  s.ensure_partial(1 << 16);
  dev::init_red_scratch(s.rs);
}

void Context::init_local(const std::vector<int>& devices) {
  if (devices.empty() || devices.size() > 16) fail(GKB_EINVAL, "gkb_init: need 1..16 shards");
  int ndev = 0;
  GKB_CUDA(cudaGetDeviceCount(&ndev));
  shards.resize(devices.size());
  for (size_t i = 0; i < devices.size(); ++i) {
    if (devices[i] < 0 || devices[i] >= ndev) fail(GKB_EINVAL, "gkb_init: bad device ordinal");
    init_shard(shards[i], (int)i, devices[i]);
  }
  nshards_total = (int)devices.size();
  first_shard = 0;
  spmd_mode = false;
}

void Context::init_nccl(int device, const ncclUniqueId& id, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GKB_EINVAL, "gkb_init_nccl: bad rank");
  shards.resize(1);
  init_shard(shards[0], rank, device);
  nshards_total = nranks;
  first_shard = rank;
  spmd_mode = true;
  GKB_CUDA(cudaSetDevice(device));
  check_nccl(ncclCommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
}

void Context::init_host(int device, int nranks, int rank, gkb_host_allreduce_fn fn, void* user) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GKB_EINVAL, "gkb_init_host_comm: bad rank");
  if (!fn) fail(GKB_EINVAL, "gkb_init_host_comm: null allreduce function");
  shards.resize(1);
  init_shard(shards[0], rank, device);
  nshards_total = nranks;
  first_shard = rank;
  spmd_mode = true;
  host_fn = fn;
  host_user = user;
}

namespace {
struct HostAllreduce {
  gkb_host_allreduce_fn fn;
  void* user;
  double* buf;
  int64_t count;
};
void CUDART_CB host_allreduce_tramp(void* p) {
  const HostAllreduce* a = static_cast<const HostAllreduce*>(p);
  a->fn(a->user, a->buf, a->count);
  delete a;
}
}  // namespace

Context::~Context() {
  for (auto& s : shards) {
    cudaSetDevice(s.dev);
    if (s.stream) cudaStreamSynchronize(s.stream);
    if (s.rs.partial) cudaFree(s.rs.partial);
    if (s.rs.ticket) cudaFree(s.rs.ticket);
    if (s.dres) cudaFree(s.dres);
    if (s.hres) cudaFreeHost(s.hres);
    for (int q = 0; q < 2; ++q)
      if (s.hstage[q]) cudaFreeHost(s.hstage[q]);
    if (s.flush_buf) cudaFree(s.flush_buf);
    if (s.ev) cudaEventDestroy(s.ev);
    if (host_buf) cudaFreeHost(host_buf);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  if (stage && !shards.empty()) {
    cudaSetDevice(shards[0].dev);
    cudaFree(stage);
  }
  if (comm) ncclCommDestroy(comm);
}

void Context::set_device(int i) const { GKB_CUDA(cudaSetDevice(shards[i].dev)); }

void Context::sync_all() {
  for (auto& s : shards) {
    GKB_CUDA(cudaSetDevice(s.dev));
    GKB_CUDA(cudaStreamSynchronize(s.stream));
  }
}

void Context::allreduce(const std::vector<double*>& bufs, int64_t count) {
  if (count == 0) return;
  if (spmd_mode) {
    // GKB_NCCL_FORCE=1 (tests): a one-rank NCCL context still calls
    // ncclAllReduce (an identity), so the NCCL path runs on a one-GPU box
    static const bool force = [] {
      const char* e = getenv("GKB_NCCL_FORCE");
      return e && e[0] == '1';
    }();
    if (nshards_total == 1 && !(force && comm && !host_fn)) return;
    Shard& s = shards[0];
    GKB_CUDA(cudaSetDevice(s.dev));
    if (host_fn) {
      // stream-ordered: the host function runs after the D2H copy and before
      // the H2D copy on the shard's stream (it must not call CUDA); one
      // staging buffer serves every call since the stream serializes them
      const size_t bytes = sizeof(double) * (size_t)count;
      if (host_cap < count) {
        GKB_CUDA(cudaStreamSynchronize(s.stream));
        if (host_buf) GKB_CUDA(cudaFreeHost(host_buf));
        host_buf = nullptr;
        host_cap = std::max<int64_t>(count, 1 << 12);
        GKB_CUDA(cudaMallocHost(&host_buf, sizeof(double) * (size_t)host_cap));
      }
      GKB_CUDA(cudaMemcpyAsync(host_buf, bufs[0], bytes, cudaMemcpyDeviceToHost, s.stream));
      GKB_CUDA(cudaLaunchHostFunc(s.stream, host_allreduce_tramp,
                                  new HostAllreduce{host_fn, host_user, host_buf, count}));
      GKB_CUDA(cudaMemcpyAsync(bufs[0], host_buf, bytes, cudaMemcpyHostToDevice, s.stream));
      return;
    }
    check_nccl(ncclAllReduce(bufs[0], bufs[0], (size_t)count, ncclDouble, ncclSum, comm, s.stream),
               "ncclAllReduce");
    return;
  }
  const int G = (int)shards.size();
  if (G == 1) return;
  // Gather every shard's buffer on shard 0's device, sum in shard order,
  // scatter the identical result back.
  Shard& s0 = shards[0];
  GKB_CUDA(cudaSetDevice(s0.dev));
  if (stage_cap < count * G) {
    if (stage) GKB_CUDA(cudaFree(stage));
    stage_cap = std::max<int64_t>(count * G, 1 << 16);
    GKB_CUDA(cudaMalloc(&stage, sizeof(double) * (size_t)stage_cap));
  }
  for (int i = 1; i < G; ++i) {
    GKB_CUDA(cudaSetDevice(shards[i].dev));
    GKB_CUDA(cudaEventRecord(shards[i].ev, shards[i].stream));
    GKB_CUDA(cudaSetDevice(s0.dev));
    GKB_CUDA(cudaStreamWaitEvent(s0.stream, shards[i].ev, 0));
  }
  GKB_CUDA(cudaSetDevice(s0.dev));
  std::vector<const double*> srcs(G);
  for (int i = 0; i < G; ++i) {
    double* dst = stage + (int64_t)i * count;
    GKB_CUDA(cudaMemcpyPeerAsync(dst, s0.dev, bufs[i], shards[i].dev, sizeof(double) * (size_t)count,
                                 s0.stream));
    srcs[i] = dst;
  }
  dev::sum_buffers(srcs.data(), G, bufs[0], count, s0.stream);
  GKB_LAUNCH_CHECK();
  for (int i = 1; i < G; ++i)
    GKB_CUDA(cudaMemcpyPeerAsync(bufs[i], shards[i].dev, bufs[0], s0.dev,
                                 sizeof(double) * (size_t)count, s0.stream));
  GKB_CUDA(cudaEventRecord(s0.ev, s0.stream));
  for (int i = 1; i < G; ++i) {
    GKB_CUDA(cudaSetDevice(shards[i].dev));
    GKB_CUDA(cudaStreamWaitEvent(shards[i].stream, s0.ev, 0));
  }
  GKB_CUDA(cudaSetDevice(s0.dev));
}

std::vector<int64_t> partition_rows(int64_t m, int nparts) {
  if (nparts < 1) fail(GKB_EINVAL, "partition_rows: nparts < 1");
  if (m < 0) fail(GKB_EINVAL, "partition_rows: negative size");
  std::vector<int64_t> st(nparts + 1);
  const int64_t quads = (m + 3) / 4;
  for (int i = 0; i <= nparts; ++i) {
    int64_t q = quads * i / nparts;
    st[i] = std::min<int64_t>(m, 4 * q);
  }
  st[nparts] = m;
  return st;
}

}  // namespace gkb
