"""Block subspace iteration on X X^T -- the reference's subspace_iterate
(/root/reference/proj/src/subspace.cpp:49-115, subspace.hpp:10-70) run on the
device operator: each gram pass is two block products (gkb_op_apply_adjoint_block
then gkb_op_apply_block: the k columns of subspace.cpp:70-77 back to back on
the GPU, one host round trip per pass), the final Rayleigh-Ritz projection one
more. The k-column host work (thin QR, condition, delta) stays on the host in
LAPACK, as in the reference (Eigen HouseholderQR / JacobiSVD).

Same names, defaults, validation messages and mvp accounting
(2k per recorded iteration, including the initial range pass, plus k).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List

import numpy as np


class SubspaceVariant(enum.IntEnum):  # subspace.hpp:13-16
    kNormalize = 0  # scale each column to unit norm (no orthogonalization)
    kQr = 1         # thin QR, sign-fixed so reruns are deterministic


@dataclass
class SubspaceState:  # subspace.hpp:21-25
    iterations: int = 0
    delta_history: List[float] = field(default_factory=list)
    invcond_history: List[float] = field(default_factory=list)


@dataclass
class SubspaceResult:  # subspace.hpp:27-35
    basis: np.ndarray
    eigvals: np.ndarray
    singvals: np.ndarray
    state: SubspaceState
    converged: bool = False
    rank_deficient: bool = False
    mvps: int = 0


@dataclass
class BasisCondition:  # subspace.hpp:45-48
    kappa: float = 0.0
    inv_kappa: float = 0.0


def qr_thin(M: np.ndarray):
    """qr_thin (orth.cpp:7-21): Householder QR, signs flipped so diag(R) >= 0."""
    Q, R = np.linalg.qr(np.asarray(M, dtype=np.float64), mode="reduced")
    s = np.where(np.diag(R) < 0.0, -1.0, 1.0)
    return Q * s[None, :], R * s[:, None]


def orthonormality_error(Q: np.ndarray) -> float:
    """orthonormality_error (orth.cpp:23-29): max |Q^T Q - I|."""
    Q = np.asarray(Q, dtype=np.float64)
    return float(np.abs(Q.T @ Q - np.eye(Q.shape[1])).max()) if Q.shape[1] else 0.0


def delta_criterion(prev: np.ndarray, curr: np.ndarray, scaled: bool = True) -> float:
    """subspace.cpp:13-21: ||curr - prev||_F (/ sqrt(rows*cols) when scaled)."""
    if prev.shape != curr.shape:
        raise ValueError("delta_criterion: shape mismatch")
    raw = float(np.sqrt(((curr - prev) ** 2).sum()))
    if not scaled:
        return raw
    return raw / np.sqrt(float(prev.shape[0]) * float(prev.shape[1]))


def basis_condition(Y: np.ndarray) -> BasisCondition:
    """subspace.cpp:23-31 (singular values of the basis)."""
    s = np.linalg.svd(np.asarray(Y, dtype=np.float64), compute_uv=False)
    smax, smin = float(s[0]), float(s[-1])
    out = BasisCondition()
    out.inv_kappa = smin / smax if smax > 0.0 else 0.0
    out.kappa = smax / smin if smin > 0.0 else float("inf")
    return out


def _renormalize(Y: np.ndarray, variant: SubspaceVariant) -> np.ndarray:
    if variant == SubspaceVariant.kQr:
        return qr_thin(Y)[0]
    Y = Y.copy()
    for j in range(Y.shape[1]):
        nrm = float(np.sqrt((Y[:, j] ** 2).sum()))
        if nrm > 0.0:
            Y[:, j] /= nrm
    return Y


def subspace_iterate(op, k: int, variant: SubspaceVariant = SubspaceVariant.kQr,
                     tol: float = 1e-8, max_iter: int = 1000, seed: int = 0,
                     scaled_delta: bool = True) -> SubspaceResult:
    """subspace_iterate (subspace.cpp:49-115). `op` provides rows(), cols(),
    apply_block(), apply_adjoint_block() and mvps() (a device operator, or a
    CPU oracle adapter in the tests)."""
    m, n = op.rows(), op.cols()
    if k <= 0 or k > min(m, n):
        raise ValueError("subspace_iterate: k out of range")
    if max_iter < 0:
        raise ValueError("subspace_iterate: max_iter must be >= 0")
    if variant == SubspaceVariant.kQr and getattr(op, "_h", None):
        res = _subspace_qr_device(op, k, tol, max_iter, seed, scaled_delta)
        if res is not None:
            return res
    from .gkl import rng_normal
    mv0 = op.mvps()
    # Y(i, j) = rng.normal(), j outer, i inner (subspace.cpp:64-66)
    Y = rng_normal(seed, m * k).reshape(k, m).T.copy()
    Y = qr_thin(Y)[0]

    def gram_apply(Z):  # Z <- X X^T Z (2k products, subspace.cpp:70-77)
        return op.apply_block(op.apply_adjoint_block(Z))

    state = SubspaceState()
    converged = False
    Y = _renormalize(gram_apply(Y), variant)  # iteration 0: initial range
    state.invcond_history.append(basis_condition(Y).inv_kappa)
    for it in range(1, max_iter + 1):
        Y_prev = Y
        Y = _renormalize(gram_apply(Y), variant)
        state.iterations = it
        state.invcond_history.append(basis_condition(Y).inv_kappa)
        delta = delta_criterion(Y_prev, Y, scaled_delta)
        state.delta_history.append(delta)
        if delta <= tol:
            converged = True
            break
    rank_deficient = state.invcond_history[-1] < 1e-12
    # Rayleigh-Ritz on span(Y): singular values of X^T Q (subspace.cpp:103-110)
    Q = Y if variant == SubspaceVariant.kQr else qr_thin(Y)[0]
    Z = op.apply_adjoint_block(Q)
    sv = np.linalg.svd(Z, compute_uv=False)
    return SubspaceResult(basis=Y, eigvals=sv ** 2, singvals=sv, state=state,
                          converged=converged, rank_deficient=rank_deficient,
                          mvps=op.mvps() - mv0)


def _subspace_qr_device(op, k, tol, max_iter, seed, scaled_delta):
    """The QR variant with the blocks resident on the device
    (gkb_subspace_qr: CholeskyQR2 renormalization, device convergence test,
    one small read-back per pass). None if the block lost rank on the way --
    the host path's Householder QR then reruns the solve."""
    import ctypes as C
    from . import _lib
    res = C.POINTER(_lib.gkb_subspace_result)()
    st = _lib.lib.gkb_subspace_qr(op._h, int(k), float(tol), int(max_iter),
                                  int(seed) & 0xFFFFFFFFFFFFFFFF, int(bool(scaled_delta)),
                                  C.byref(res))
    if st != 0:
        if st == _lib.GKB_ELOGIC and "lost rank" in _lib.lib.gkb_last_error().decode():
            return None
        _lib.check(st)
    try:
        r = res.contents
        m, it = int(r.m), int(r.iterations)

        def arr(p, cnt):
            return np.ctypeslib.as_array(p, shape=(cnt,)).copy() if cnt > 0 else np.zeros(0)

        basis = np.ctypeslib.as_array(r.basis, shape=(k, m)).T.copy(order="F")
        state = SubspaceState(iterations=it,
                              delta_history=[float(v) for v in arr(r.delta_history, it)],
                              invcond_history=[float(v) for v in arr(r.invcond_history, it + 1)])
        return SubspaceResult(basis=basis, eigvals=arr(r.eigvals, k), singvals=arr(r.singvals, k),
                              state=state, converged=bool(r.converged),
                              rank_deficient=bool(r.rank_deficient), mvps=int(r.mvps))
    finally:
        _lib.lib.gkb_subspace_result_free(res)
