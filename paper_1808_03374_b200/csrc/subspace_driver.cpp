// subspace_iterate (reference /root/reference/proj/src/subspace.cpp:49-115),
// QR variant, with the k-column blocks resident on the device.
//
// The reference renormalizes Y (m x k) by a Householder thin QR with signs
// fixed so diag(R) >= 0 (orth.cpp:7-21) and measures the basis condition by a
// JacobiSVD of Y (subspace.cpp:23-31). Here Y stays in HBM (sharded by rows
// like the Lanczos U basis) and the QR is CholeskyQR2: G = W^T W on the device
// (one fixed-order reduction per column, summed across shards), R = chol(G)
// on the host (k x k), W <- W R^-1 on the device, once more for
// orthogonality. Cholesky's R has a positive diagonal, so Q is the same
// sign-fixed factor up to rounding. The condition of the orthonormal Q follows
// from the second pass on the host (Q^T Q = R2^-T G2 R2^-1). The gram pass
// X X^T is a k-column adjoint + apply block (two columns per pass on the
// genotype operator); the convergence test
// ||Y - Y_prev||_F is a device reduction. Per iteration the host reads two
// k x k Gram matrices and one scalar.
//
// Used for ScalingScheme-independent device operators when the variant is
// kQr; the kNormalize variant (whose rank-deficiency test needs the exact
// singular values of an ill-conditioned Y) runs through the host path
// (paper_1808_03374_b200/subspace.py).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "host.hpp"

namespace gkb {

namespace {

// Cholesky of the k x k symmetric G (column-major): G = R^T R, R upper with a
// positive diagonal. false if G is not numerically positive definite.
bool cholesky_upper(const std::vector<double>& G, int64_t k, std::vector<double>& R) {
  R.assign((size_t)(k * k), 0.0);
  for (int64_t j = 0; j < k; ++j) {
    double d = G[j + j * k];
    for (int64_t l = 0; l < j; ++l) d -= R[l + j * k] * R[l + j * k];
    if (!(d > 0.0)) return false;
    const double rjj = std::sqrt(d);
    R[j + j * k] = rjj;
    for (int64_t c = j + 1; c < k; ++c) {
      double s = G[j + c * k];
      for (int64_t l = 0; l < j; ++l) s -= R[l + j * k] * R[l + c * k];
      R[j + c * k] = s / rjj;
    }
  }
  return true;
}

// inverse of an upper-triangular k x k matrix (column-major)
std::vector<double> inv_upper(const std::vector<double>& R, int64_t k) {
  std::vector<double> X((size_t)(k * k), 0.0);
  for (int64_t j = 0; j < k; ++j) {
    X[j + j * k] = 1.0 / R[j + j * k];
    for (int64_t i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int64_t l = i + 1; l <= j; ++l) s += R[i + l * k] * X[l + j * k];
      X[i + j * k] = -s / R[i + i * k];
    }
  }
  return X;
}

// sqrt(lambda_min / lambda_max) of a small symmetric PSD matrix (cyclic Jacobi)
double inv_cond_from_gram(std::vector<double> A, int64_t k) {
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int64_t p = 0; p < k; ++p)
      for (int64_t q = p + 1; q < k; ++q) off += A[p + q * k] * A[p + q * k];
    if (off < 1e-300) break;
    for (int64_t p = 0; p < k; ++p)
      for (int64_t q = p + 1; q < k; ++q) {
        const double apq = A[p + q * k];
        if (apq == 0.0) continue;
        const double theta = (A[q + q * k] - A[p + p * k]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::hypot(1.0, theta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
        for (int64_t r = 0; r < k; ++r) {  // A <- A J
          const double x = A[r + p * k], y = A[r + q * k];
          A[r + p * k] = c * x - s * y;
          A[r + q * k] = s * x + c * y;
        }
        for (int64_t r = 0; r < k; ++r) {  // A <- J^T A
          const double x = A[p + r * k], y = A[q + r * k];
          A[p + r * k] = c * x - s * y;
          A[q + r * k] = s * x + c * y;
        }
      }
  }
  double lo = A[0], hi = A[0];
  for (int64_t i = 1; i < k; ++i) {
    lo = std::min(lo, A[i + i * k]);
    hi = std::max(hi, A[i + i * k]);
  }
  if (!(hi > 0.0)) return 0.0;
  return lo > 0.0 ? std::sqrt(lo / hi) : 0.0;
}

}  // namespace

SubspaceOutput subspace_qr_device(DevOp* op, int64_t k, double tol, int64_t max_iter,
                                  uint64_t seed, bool scaled_delta) {
  const int64_t m = op->m, n = op->n;
  if (k <= 0 || k > std::min(m, n)) fail(GKB_EINVAL, "subspace_iterate: k out of range");
  if (max_iter < 0) fail(GKB_EINVAL, "subspace_iterate: max_iter must be >= 0");
  Context* ctx = op->ctx;
  const int L = (int)ctx->shards.size();
  std::vector<double*> Y(L), W(L), Z(L), Wk(L);
  std::vector<int64_t> r(L);
  for (int i = 0; i < L; ++i) {
    ctx->set_device(i);
    cudaStream_t st = ctx->shards[i].stream;
    r[i] = op->rows(i);
    const size_t rk = (size_t)std::max<int64_t>(r[i] * k, 1);
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&Y[i]), sizeof(double) * rk, st));
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&W[i]), sizeof(double) * rk, st));
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&Z[i]), sizeof(double) * (size_t)(n * k), st));
    GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&Wk[i]), sizeof(double) * (size_t)(k * k), st));
    ctx->shards[i].ensure_partial(dev::red_blocks(std::max<int64_t>(r[i], 1)) * (k + 2) + 64);
  }
  auto release = [&]() {
    for (int i = 0; i < L; ++i) {
      ctx->set_device(i);
      cudaStream_t st = ctx->shards[i].stream;
      for (double* p : {Y[i], W[i], Z[i], Wk[i]})
        if (p) cudaFreeAsync(p, st);
      cudaStreamSynchronize(st);
    }
  };
  SubspaceOutput out;
  try {
    // k x k Gram of the block B (rows(i) x k per shard), summed across shards
    for (int i = 0; i < L; ++i) ctx->shards[i].ensure_res(k * k + 64);
    auto gram = [&](const std::vector<double*>& B) {
      for (int i = 0; i < L; ++i) {
        ctx->set_device(i);
        Shard& sh = ctx->shards[i];
        for (int64_t j = 0; j < k; ++j)
          dev::gemv_t(B[i], std::max<int64_t>(r[i], 1), r[i], k, B[i] + j * r[i], false, sh.rs,
                      sh.dres + j * k, sh.stream);
      }
      std::vector<double*> b(L);
      for (int i = 0; i < L; ++i) b[i] = ctx->shards[i].dres;
      ctx->allreduce(b, k * k);
      ctx->set_device(0);
      Shard& s0 = ctx->shards[0];
      std::vector<double> G((size_t)(k * k));
      GKB_CUDA(cudaMemcpyAsync(s0.hres, s0.dres, sizeof(double) * (size_t)(k * k),
                               cudaMemcpyDeviceToHost, s0.stream));
      ctx->sync_all();
      std::copy(s0.hres, s0.hres + k * k, G.begin());
      for (int64_t a = 0; a < k; ++a)  // symmetrize (the two triangles are separate sums)
        for (int64_t c = a + 1; c < k; ++c) {
          const double v = 0.5 * (G[a + c * k] + G[c + a * k]);
          G[a + c * k] = G[c + a * k] = v;
        }
      return G;
    };
    // dst <- src * M (M host k x k)
    auto times = [&](const std::vector<double*>& src, const std::vector<double>& M,
                     const std::vector<double*>& dst) {
      for (int i = 0; i < L; ++i) {
        ctx->set_device(i);
        cudaStream_t st = ctx->shards[i].stream;
        GKB_CUDA(cudaMemcpyAsync(Wk[i], M.data(), sizeof(double) * (size_t)(k * k),
                                 cudaMemcpyHostToDevice, st));
        dev::gemm_small(src[i], std::max<int64_t>(r[i], 1), r[i], k, Wk[i], k, k, dst[i],
                        std::max<int64_t>(r[i], 1), st);
        GKB_CUDA(cudaStreamSynchronize(st));  // M is a host temporary
      }
    };
    // W (raw block) -> Y (orthonormal, diag(R) > 0); returns inv_kappa of Y
    auto renormalize = [&]() -> double {
      std::vector<double> R;
      std::vector<double> G1 = gram(W);
      if (!cholesky_upper(G1, k, R))
        fail(GKB_ELOGIC, "subspace_iterate: basis lost rank (Cholesky QR); use the host path");
      times(W, inv_upper(R, k), Y);  // Y = W R1^-1
      std::vector<double> G2 = gram(Y), R2;
      if (!cholesky_upper(G2, k, R2))
        fail(GKB_ELOGIC, "subspace_iterate: basis lost rank (Cholesky QR); use the host path");
      const std::vector<double> R2i = inv_upper(R2, k);
      times(Y, R2i, W);  // W = Y R2^-1 = Q
      std::swap(Y, W);
      // Q^T Q = R2^-T G2 R2^-1
      std::vector<double> T((size_t)(k * k), 0.0), QtQ((size_t)(k * k), 0.0);
      for (int64_t a = 0; a < k; ++a)
        for (int64_t c = 0; c < k; ++c) {
          double s = 0.0;
          for (int64_t l = 0; l < k; ++l) s += G2[a + l * k] * R2i[l + c * k];
          T[a + c * k] = s;
        }
      for (int64_t a = 0; a < k; ++a)
        for (int64_t c = 0; c < k; ++c) {
          double s = 0.0;
          for (int64_t l = 0; l < k; ++l) s += R2i[l + a * k] * T[l + c * k];
          QtQ[a + c * k] = s;
        }
      return inv_cond_from_gram(QtQ, k);
    };
    int64_t mvps = 0;
    // X X^T on the block Y -> W, column by column (subspace.cpp:70-77)
    // (block products: the operator may take several columns per pass)
    auto gram_apply = [&]() {
      std::vector<const double*> yin(L), zin(L);
      std::vector<double*> zout(L), wout(L);
      for (int i = 0; i < L; ++i) {
        yin[i] = Y[i];
        zout[i] = Z[i];
        zin[i] = Z[i];
        wout[i] = W[i];
      }
      op->adjoint_block_dev(yin, r, k, zout, n);
      op->apply_block_dev(zin, n, k, wout, r);
      mvps += 2 * k;
    };

    // start: Y(i, j) = rng.normal(), j outer, i inner (subspace.cpp:64-66), then QR
    {
      Rng rng(seed);
      std::vector<double> Yh((size_t)(m * k));
      for (auto& v : Yh) v = rng.normal();
      for (int i = 0; i < L; ++i) {
        ctx->set_device(i);
        if (r[i] > 0)
          GKB_CUDA(cudaMemcpy2DAsync(W[i], sizeof(double) * (size_t)r[i], Yh.data() + op->row0(i),
                                     sizeof(double) * (size_t)m, sizeof(double) * (size_t)r[i],
                                     (size_t)k, cudaMemcpyHostToDevice, ctx->shards[i].stream));
      }
      ctx->sync_all();
      renormalize();
    }
    // iteration 0: initial range
    gram_apply();
    out.invcond_history.push_back(renormalize());
    std::vector<double*> Yprev(L);
    for (int i = 0; i < L; ++i) {
      ctx->set_device(i);
      GKB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&Yprev[i]),
                               sizeof(double) * (size_t)std::max<int64_t>(r[i] * k, 1),
                               ctx->shards[i].stream));
    }
    for (int64_t it = 1; it <= max_iter; ++it) {
      for (int i = 0; i < L; ++i) {
        ctx->set_device(i);
        if (r[i] > 0)
          GKB_CUDA(cudaMemcpyAsync(Yprev[i], Y[i], sizeof(double) * (size_t)(r[i] * k),
                                   cudaMemcpyDeviceToDevice, ctx->shards[i].stream));
      }
      gram_apply();
      out.invcond_history.push_back(renormalize());
      out.iterations = it;
      // ||Y - Y_prev||_F (delta_criterion, subspace.cpp:13-21)
      for (int i = 0; i < L; ++i) {
        ctx->set_device(i);
        Shard& sh = ctx->shards[i];
        dev::diff_nrm2sq(Y[i], Yprev[i], r[i] * k, sh.rs, sh.dres, sh.stream);
      }
      std::vector<double*> b(L);
      for (int i = 0; i < L; ++i) b[i] = ctx->shards[i].dres;
      ctx->allreduce(b, 1);
      ctx->set_device(0);
      Shard& s0 = ctx->shards[0];
      GKB_CUDA(cudaMemcpyAsync(s0.hres, s0.dres, sizeof(double), cudaMemcpyDeviceToHost,
                               s0.stream));
      ctx->sync_all();
      double delta = std::sqrt(s0.hres[0]);
      if (scaled_delta) delta /= std::sqrt(static_cast<double>(m) * static_cast<double>(k));
      out.delta_history.push_back(delta);
      if (delta <= tol) {
        out.converged = true;
        break;
      }
    }
    for (int i = 0; i < L; ++i) {
      ctx->set_device(i);
      cudaFreeAsync(Yprev[i], ctx->shards[i].stream);
    }
    out.rank_deficient = out.invcond_history.back() < 1e-12;
    // Rayleigh-Ritz: singular values of X^T Q (subspace.cpp:103-110)
    {
      std::vector<const double*> yin(L);
      std::vector<double*> zout(L);
      for (int i = 0; i < L; ++i) {
        yin[i] = Y[i];
        zout[i] = Z[i];
      }
      op->adjoint_block_dev(yin, r, k, zout, n);
    }
    mvps += k;
    std::vector<double> Zh((size_t)(n * k));
    ctx->set_device(0);
    GKB_CUDA(cudaMemcpyAsync(Zh.data(), Z[0], sizeof(double) * (size_t)(n * k),
                             cudaMemcpyDeviceToHost, ctx->shards[0].stream));
    ctx->sync_all();
    std::vector<double> U((size_t)(n * k)), V((size_t)(k * k));
    out.singvals.assign((size_t)k, 0.0);
    svd_small(Zh.data(), n, k, U.data(), out.singvals.data(), V.data());
    out.eigvals.resize((size_t)k);
    for (int64_t i = 0; i < k; ++i) out.eigvals[i] = out.singvals[i] * out.singvals[i];
    // basis (m x k, column-major) from the row shards
    out.basis.assign((size_t)(m * k), 0.0);
    if (ctx->spmd_mode && ctx->nshards_total > 1) {
      ctx->set_device(0);
      Shard& s = ctx->shards[0];
      double* full = nullptr;
      GKB_CUDA(cudaMalloc(&full, sizeof(double) * (size_t)(m * k)));
      GKB_CUDA(cudaMemsetAsync(full, 0, sizeof(double) * (size_t)(m * k), s.stream));
      if (r[0] > 0)
        GKB_CUDA(cudaMemcpy2DAsync(full + op->row0(0), sizeof(double) * (size_t)m, Y[0],
                                   sizeof(double) * (size_t)r[0], sizeof(double) * (size_t)r[0],
                                   (size_t)k, cudaMemcpyDeviceToDevice, s.stream));
      ctx->allreduce({full}, m * k);
      GKB_CUDA(cudaMemcpyAsync(out.basis.data(), full, sizeof(double) * (size_t)(m * k),
                               cudaMemcpyDeviceToHost, s.stream));
      GKB_CUDA(cudaStreamSynchronize(s.stream));
      cudaFree(full);
    } else {
      for (int i = 0; i < L; ++i) {
        ctx->set_device(i);
        if (r[i] > 0)
          GKB_CUDA(cudaMemcpy2DAsync(out.basis.data() + op->row0(i), sizeof(double) * (size_t)m,
                                     Y[i], sizeof(double) * (size_t)r[i],
                                     sizeof(double) * (size_t)r[i], (size_t)k,
                                     cudaMemcpyDeviceToHost, ctx->shards[i].stream));
      }
      ctx->sync_all();
    }
    out.mvps = mvps;
    op->mvps += mvps;
  } catch (...) {
    release();
    throw;
  }
  release();
  return out;
}

}  // namespace gkb
