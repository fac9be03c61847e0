"""PC-adjusted marker regression -- the reference's ols_fit / pc_adjusted_fit
(/root/reference/proj/src/regress.cpp:10-65) and the per-marker scan of
`gkpca regress` (tools/gkpca.cpp:554-680), with the scan's data pass on the
device.

The scan fits, for every marker i, y ~ [1, m_i, Z] (Z = sample-side principal
components). The reference refactors that (n x (k+2)) design for each marker;
here all markers share one device pass: the block product of the operator
with [y, 1, Z] (gkb_op_apply_block, k+2 columns) gives m_i.y, m_i.1 and m_i.Z,
m_i.m_i comes from the marker counts, and the per-marker coefficients follow
by partialling out C = [1, Z] (Frisch-Waugh-Lovell):
    d_i   = m_i.m_i - u_i' A^-1 u_i,        u_i = C' m_i, A = C'C
    beta  = (m_i.y - u_i' A^-1 w) / d_i,    w = C'y
    RSS   = (y.y - w' A^-1 w) - beta^2 d_i
    sigma2 = RSS / (n or n - (k+2)),  se = sqrt(sigma2 / d_i)
    [intercept, gamma] = A^-1 (w - u_i beta)
-- the same estimates as the reference's QR solve. A marker that is constant
(fewer than two distinct values after mean imputation) is reported with the
reference's rank-deficiency error for design column 1.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

EPS = np.finfo(np.float64).eps


class RankDeficiencyError(RuntimeError):
    """regress.hpp:12-19: `column` names the first dependent design column."""

    def __init__(self, column: int, what: str):
        super().__init__(what)
        self.column = column


@dataclass
class RegressionResult:  # regress.hpp:23-28
    beta_hat: np.ndarray
    sigma2_hat: float
    cov_beta: np.ndarray
    residuals: np.ndarray


@dataclass
class PcAdjustedResult:  # regress.hpp:39-44
    joint: RegressionResult
    beta_hat: np.ndarray
    gamma_hat: np.ndarray
    cov_beta: np.ndarray


def ols_fit(X, y, unbiased: bool = False) -> RegressionResult:
    """ols_fit (regress.cpp:10-43): thin QR (sign-fixed), |R_ii| <= max|R_jj| *
    max(n, p) * eps flags column i, beta = R^-1 Q'y, cov = sigma2 R^-1 R^-T."""
    from .subspace import qr_thin
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).ravel()
    if X.ndim == 1:
        X = X[:, None]
    n, p = X.shape
    if y.size != n:
        raise ValueError("ols_fit: y length does not match rows of X")
    if p == 0 or n < p:
        raise ValueError("ols_fit: need 0 < cols <= rows")
    Q, R = qr_thin(X)
    d = np.abs(np.diag(R))
    tol = d.max() * max(n, p) * EPS
    for i in range(p):
        if d[i] <= tol:
            raise RankDeficiencyError(
                i, f"ols_fit: design column {i} is linearly dependent on earlier columns")
    beta = np.linalg.solve(np.triu(R), Q.T @ y)
    res = y - X @ beta
    denom = float(n - p) if unbiased else float(n)
    sigma2 = float(res @ res) / denom
    rinv = np.linalg.solve(np.triu(R), np.eye(p))
    return RegressionResult(beta, sigma2, sigma2 * (rinv @ rinv.T), res)


def pc_adjusted_fit(X, Z, y, unbiased: bool = False) -> PcAdjustedResult:
    """pc_adjusted_fit (regress.cpp:45-63): joint fit of y on [X Z]."""
    X = np.asarray(X, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    if Z.ndim == 1:
        Z = Z[:, None]
    if Z.shape[0] != X.shape[0]:
        raise ValueError("pc_adjusted_fit: Z rows do not match X")
    p = X.shape[1]
    joint = ols_fit(np.hstack([X, Z]), y, unbiased)
    return PcAdjustedResult(joint, joint.beta_hat[:p], joint.beta_hat[p:],
                            joint.cov_beta[:p, :p])


@dataclass
class MarkerScan:
    beta: np.ndarray
    se: np.ndarray
    intercept: np.ndarray
    sigma2: np.ndarray
    dependent: np.ndarray  # bool: reported as RankDeficiencyError(column 1)


def marker_sumsq(op) -> np.ndarray:
    """sum_s x_is^2 of every row of a genotype operator, from its counts and
    scaling: inv_s^2 [n0 mu^2 + n1 (1-mu)^2 + n2 (2-mu)^2 + nmiss (mean-mu)^2]."""
    c = op.counts().astype(np.float64)
    mu, inv_s = op.scaling()
    obs = c[:, 0] + c[:, 1] + c[:, 2]
    mean = np.where(obs > 0, (c[:, 1] + 2 * c[:, 2]) / np.maximum(obs, 1), 0.0)
    ss = (c[:, 0] * mu ** 2 + c[:, 1] * (1 - mu) ** 2 + c[:, 2] * (2 - mu) ** 2
          + c[:, 3] * (mean - mu) ** 2)
    return ss * inv_s ** 2


def constant_markers(op) -> np.ndarray:
    """Markers whose row is constant (fewer than two distinct values after
    impute_mean): zero variance, or one observed dosage whose value the
    imputed entries repeat. With an intercept such a column is dependent."""
    c = op.counts()
    distinct = (c[:, 0] > 0).astype(int) + (c[:, 1] > 0) + (c[:, 2] > 0)
    _, inv_s = op.scaling()
    return (distinct < 2) | (inv_s == 0.0)


def marker_scan(op, y, Z: Optional[np.ndarray] = None, unbiased: bool = False,
                sumsq: Optional[np.ndarray] = None,
                constant: Optional[np.ndarray] = None) -> MarkerScan:
    """Per-marker fits of y ~ [1, m_i, Z] for every row m_i of `op` (rows x n):
    one block product op.apply_block([y, 1, Z]) plus O(rows k^2) host algebra."""
    y = np.asarray(y, dtype=np.float64).ravel()
    n = op.cols()
    if y.size != n:
        raise ValueError("marker_scan: phenotype length does not match samples")
    if sumsq is None and constant is None and hasattr(op, "marker_scan"):
        # genotype operator: block product and per-marker algebra on the device
        try:
            beta, se, icpt, s2, dep = op.marker_scan(y, Z, unbiased)
            return MarkerScan(beta, se, icpt, s2, dep)
        except Exception as e:  # SPMD operators keep the host algebra
            if "SPMD" not in str(e):
                raise
    Zm = np.zeros((n, 0)) if Z is None else np.asarray(Z, dtype=np.float64).reshape(n, -1)
    C = np.hstack([np.ones((n, 1)), Zm])                    # shared nuisance columns
    P = op.apply_block(np.hstack([y[:, None], C]))          # [m.y, m.1, m.Z] per marker
    my, U = P[:, 0], P[:, 1:]
    q = marker_sumsq(op) if sumsq is None else np.asarray(sumsq, dtype=np.float64)
    A = C.T @ C
    Ainv = np.linalg.inv(A)
    w = C.T @ y
    AU = U @ Ainv                                           # u_i' A^-1 (rows)
    d = q - np.einsum("ij,ij->i", AU, U)
    yy_c = float(y @ y - w @ Ainv @ w)
    with np.errstate(divide="ignore", invalid="ignore"):   # dependent markers: d ~ 0
        beta = (my - AU @ w) / d
        rss = yy_c - beta ** 2 * d
        kk = C.shape[1] + 1
        denom = float(n - kk) if unbiased else float(n)
        sigma2 = rss / denom
        se = np.sqrt(sigma2 / d)
    # [A^-1 (w - u_i beta_i)]_0 = (A^-1 w)_0 - beta_i (u_i' A^-1)_0  (A^-1 symmetric)
    intercept = float(Ainv[0] @ w) - beta * AU[:, 0]
    dep = constant_markers(op) if constant is None else np.asarray(constant, dtype=bool)
    dep = dep | ~(d > 0)
    return MarkerScan(beta, se, intercept, sigma2, dep)


def scan_entries(scan: MarkerScan) -> List[dict]:
    """regression.json "markers" entries (gkpca.cpp:620-668)."""
    out = []
    for i in range(scan.beta.size):
        if scan.dependent[i]:
            out.append({"marker": i, "column": 1,
                        "error": "ols_fit: design column 1 is linearly dependent on earlier "
                                 "columns"})
        else:
            out.append({"marker": i, "beta": float(scan.beta[i]), "se": float(scan.se[i]),
                        "intercept": float(scan.intercept[i]), "sigma2": float(scan.sigma2[i])})
    return out
