"""ctypes wrapper of the CPU oracle (oracle/gkb_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product package.
The oracle restates the reference's algorithm (see gkb_oracle.h for the
file:line map) and is pinned on the reference's known-answer tests.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")


def build() -> None:
    subprocess.run(["make", "-C", HERE], check=True, stdout=subprocess.DEVNULL)


if not os.path.exists(LIB):
    build()
_o = C.CDLL(LIB)

PD = C.POINTER(C.c_double)
PU8 = C.POINTER(C.c_uint8)
PI64 = C.POINTER(C.c_int64)


class orc_gkl_options(C.Structure):
    _fields_ = [("k", C.c_int64), ("tol", C.c_double), ("max_mvps", C.c_int64),
                ("reorth", C.c_int), ("omega", C.c_double), ("one_sided", C.c_int),
                ("restart", C.c_int), ("max_subspace", C.c_int64), ("keep", C.c_int64),
                ("seed", C.c_uint64), ("record_history", C.c_int), ("omega_recurrence", C.c_int)]


class orc_op(C.Structure):
    pass


APPLY_FN = C.CFUNCTYPE(None, C.POINTER(orc_op), PD, PD)
orc_op._fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("ctx", C.c_void_p),
                   ("apply", APPLY_FN), ("apply_adjoint", APPLY_FN)]


class orc_geno(C.Structure):
    _fields_ = [("payload", PU8), ("p", C.c_int64), ("n", C.c_int64), ("stride", C.c_int64),
                ("mu", PD), ("inv_s", PD), ("nthreads", C.c_int), ("mean", PD)]


class orc_svdl_result(C.Structure):
    _fields_ = [("count", C.c_int64), ("singvals", PD), ("U", PD), ("V", PD), ("err", PD),
                ("converged", C.POINTER(C.c_int)), ("mvps", C.c_long), ("steps", C.c_int64),
                ("restarts", C.c_int), ("reorth_count", C.c_int), ("deflations", C.c_int),
                ("all_converged", C.c_int), ("wall_seconds", C.c_double),
                ("history_len", C.c_int64), ("ritz_history", PD), ("err_history", PD)]


class orc_lanczos(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("cap", C.c_int64), ("j", C.c_int64),
                ("U", PD), ("V", PD), ("B", PD), ("coupling", PD), ("mu", PD), ("nu", PD),
                ("mu_next", PD), ("nu_next", PD), ("right_exhausted", C.c_int)]


class orc_step_info(C.Structure):
    _fields_ = [("status", C.c_int), ("reorthogonalized_left", C.c_int),
                ("reorthogonalized_right", C.c_int), ("alpha", C.c_double), ("beta", C.c_double)]


class orc_ritz(C.Structure):
    _fields_ = [("j", C.c_int64), ("values", PD), ("WL", PD), ("WR", PD), ("err", PD),
                ("err_crude", PD), ("converged", C.POINTER(C.c_int))]


class orc_rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int), ("spare", C.c_double),
                ("have_spare", C.c_int)]


class orc_synth_spec(C.Structure):
    _fields_ = [("p", C.c_int64), ("n", C.c_int64), ("seed", C.c_uint64), ("npop", C.c_int),
                ("freq", PD), ("pop", C.POINTER(C.c_int32)), ("admix", PD),
                ("missing_rate", C.c_double), ("copy_from", C.POINTER(C.c_int32)),
                ("copy_prob", C.c_double)]


def _sig(name, res, args):
    f = getattr(_o, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("orc_rng_init", None, [C.POINTER(orc_rng), C.c_uint64])
_sig("orc_rng_bits", C.c_uint64, [C.POINTER(orc_rng)])
_sig("orc_rng_uniform", C.c_double, [C.POINTER(orc_rng)])
_sig("orc_rng_uniform_symmetric", C.c_double, [C.POINTER(orc_rng)])
_sig("orc_rng_uniform_int", C.c_uint64, [C.POINTER(orc_rng), C.c_uint64, C.c_uint64])
_sig("orc_rng_normal", C.c_double, [C.POINTER(orc_rng)])
_sig("orc_rng_fill_symmetric", None, [C.c_uint64, C.c_int64, PD])
_sig("orc_gaussian_matrix", None, [C.c_int64, C.c_int64, C.c_uint64, PD])
_sig("orc_bed_decode", None, [PU8, C.c_int64, C.c_int64, PU8])
_sig("orc_bed_encode", None, [PU8, C.c_int64, C.c_int64, PU8])
_sig("orc_marker_counts", None, [PU8, C.c_int64, C.c_int64, PI64])
_sig("orc_marker_scaling", None, [PI64, C.c_int64, C.c_int64, C.c_int, PD, PD])
_sig("orc_marker_means", None, [PI64, C.c_int64, PD])
_sig("orc_dense_op", None, [C.POINTER(orc_op), PD, C.c_int64, C.c_int64])
_sig("orc_geno_op", None, [C.POINTER(orc_op), C.POINTER(orc_geno)])
_sig("orc_geno_apply", None, [C.POINTER(orc_geno), PD, PD])
_sig("orc_geno_apply_adjoint", None, [C.POINTER(orc_geno), PD, PD])
_sig("orc_geno_apply_rows", None, [C.POINTER(orc_geno), C.c_int64, C.c_int64, PD, PD])
_sig("orc_geno_apply_adjoint_rows", None, [C.POINTER(orc_geno), C.c_int64, C.c_int64, PD, PD])
_sig("orc_norm_estimate", C.c_double, [C.POINTER(orc_op), C.c_int, C.c_uint64])
_sig("orc_adjoint_mismatch", C.c_double, [C.POINTER(orc_op), C.c_uint64])
_sig("orc_cgs2", C.c_double, [PD, C.c_int64, C.c_int64, PD, PD])
_sig("orc_svd_small", C.c_int, [PD, C.c_int64, C.c_int64, PD, PD, PD])
_sig("orc_gkl_options_default", None, [C.POINTER(orc_gkl_options)])
_sig("orc_gkl_options_validate", C.c_int,
     [C.POINTER(orc_gkl_options), C.c_int64, C.c_int64, C.c_char_p, C.c_size_t])
_sig("orc_lanczos_init", C.c_int, [C.POINTER(orc_lanczos), C.c_int64, C.c_int64, C.c_int64, PD])
_sig("orc_lanczos_free", None, [C.POINTER(orc_lanczos)])
_sig("orc_bidiag_step", C.c_int, [C.POINTER(orc_op), C.POINTER(orc_lanczos),
                                  C.POINTER(orc_gkl_options), C.POINTER(orc_rng), C.c_double,
                                  C.POINTER(C.c_long), C.POINTER(orc_step_info)])
_sig("orc_ritz_extract", C.c_int, [C.POINTER(orc_lanczos), C.c_double, C.POINTER(orc_ritz)])
_sig("orc_ritz_free", None, [C.POINTER(orc_ritz)])
_sig("orc_thick_restart", C.c_int, [C.POINTER(orc_lanczos), C.c_int64])
_sig("orc_compress_exhausted", None, [C.POINTER(orc_lanczos)])
_sig("orc_deflate_right", None, [C.POINTER(orc_lanczos), C.POINTER(orc_rng)])
_sig("orc_error_metric_l1", C.c_double, [C.POINTER(orc_ritz), C.c_int64])
_sig("orc_svdl", C.c_int, [C.POINTER(orc_op), C.POINTER(orc_gkl_options),
                           C.POINTER(orc_svdl_result), C.c_char_p, C.c_size_t])
_sig("orc_svdl_result_free", None, [C.POINTER(orc_svdl_result)])
_sig("orc_synth_bed", None, [C.POINTER(orc_synth_spec), C.c_int64, C.c_int64, PU8])


def _pd(a):
    return a.ctypes.data_as(PD)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ------------------------------------------------------------------ Rng
class Rng:
    def __init__(self, seed: int):
        self._r = orc_rng()
        _o.orc_rng_init(C.byref(self._r), int(seed) & 0xFFFFFFFFFFFFFFFF)

    def bits(self):
        return _o.orc_rng_bits(C.byref(self._r))

    def uniform(self):
        return _o.orc_rng_uniform(C.byref(self._r))

    def uniform_symmetric(self):
        return _o.orc_rng_uniform_symmetric(C.byref(self._r))

    def uniform_int(self, lo, hi):
        return _o.orc_rng_uniform_int(C.byref(self._r), lo, hi)

    def normal(self):
        return _o.orc_rng_normal(C.byref(self._r))


def rng_fill_symmetric(seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    _o.orc_rng_fill_symmetric(int(seed) & 0xFFFFFFFFFFFFFFFF, n, _pd(out))
    return out


def gaussian_matrix(m: int, n: int, seed: int) -> np.ndarray:
    """oracles::gaussian_matrix (tests/oracles.hpp:157-163), column-major fill."""
    out = np.empty(m * n)
    _o.orc_gaussian_matrix(m, n, int(seed), _pd(out))
    return out.reshape(n, m).T.copy()


# ------------------------------------------------------------------ genotypes
def bed_decode(payload, p, n):
    buf = np.ascontiguousarray(payload, dtype=np.uint8)
    out = np.empty(p * n, dtype=np.uint8)
    _o.orc_bed_decode(buf.ctypes.data_as(PU8), p, n, out.ctypes.data_as(PU8))
    return out.reshape(p, n)


def bed_encode(dosages):
    d = np.ascontiguousarray(dosages, dtype=np.uint8)
    p, n = d.shape
    out = np.empty(p * ((n + 3) // 4), dtype=np.uint8)
    _o.orc_bed_encode(d.ctypes.data_as(PU8), p, n, out.ctypes.data_as(PU8))
    return out


def marker_counts(payload, p, n):
    buf = np.ascontiguousarray(payload, dtype=np.uint8)
    out = np.empty(p * 4, dtype=np.int64)
    _o.orc_marker_counts(buf.ctypes.data_as(PU8), p, n, out.ctypes.data_as(PI64))
    return out.reshape(p, 4)


def marker_scaling(counts, n, scheme):
    c = np.ascontiguousarray(counts, dtype=np.int64).reshape(-1, 4)
    p = c.shape[0]
    mu, inv_s = np.empty(p), np.empty(p)
    _o.orc_marker_scaling(c.ctypes.data_as(PI64), p, n, int(scheme), _pd(mu), _pd(inv_s))
    return mu, inv_s


def marker_means(counts):
    """Observed mean per marker (0 when all missing, genio.cpp:139)."""
    c = np.ascontiguousarray(counts, dtype=np.int64).reshape(-1, 4)
    mean = np.empty(c.shape[0])
    _o.orc_marker_means(c.ctypes.data_as(PI64), c.shape[0], _pd(mean))
    return mean


class GenoOracle:
    """Packed standardized operator on the CPU (keeps its buffers alive)."""

    def __init__(self, payload, p, n, mu, inv_s, nthreads: int = 1):
        self.payload = np.ascontiguousarray(payload, dtype=np.uint8)
        self.mu, self.inv_s = _f64(mu), _f64(inv_s)
        # observed means: the value impute_mean gives a missing entry (genio.cpp:144)
        self.mean = marker_means(marker_counts(self.payload, p, n))
        self.g = orc_geno(self.payload.ctypes.data_as(PU8), p, n, (n + 3) // 4, _pd(self.mu),
                          _pd(self.inv_s), int(nthreads), _pd(self.mean))
        self.op = orc_op()
        _o.orc_geno_op(C.byref(self.op), C.byref(self.g))
        self.p, self.n = p, n

    def set_threads(self, t: int):
        self.g.nthreads = int(t)

    def apply(self, x):
        x = _f64(x)
        y = np.empty(self.p)
        _o.orc_geno_apply(C.byref(self.g), _pd(x), _pd(y))
        return y

    def apply_adjoint(self, y):
        y = _f64(y)
        z = np.empty(self.n)
        _o.orc_geno_apply_adjoint(C.byref(self.g), _pd(y), _pd(z))
        return z

    def apply_rows(self, j0, j1, x):
        x = _f64(x)
        y = np.empty(j1 - j0)
        _o.orc_geno_apply_rows(C.byref(self.g), j0, j1, _pd(x), _pd(y))
        return y

    def apply_adjoint_rows(self, j0, j1, y):
        y = _f64(y)
        z = np.empty(self.n)
        _o.orc_geno_apply_adjoint_rows(C.byref(self.g), j0, j1, _pd(y), _pd(z))
        return z


def dense_standardized(payload, p, n, mu, inv_s) -> np.ndarray:
    """The reference's literal preprocessing (load_matrix, gkpca.cpp:89-108):
    .bed decode (genio.cpp:33,53-83) -> impute_mean (missing -> observed
    row mean, genio.cpp:124-148) -> affine standardization with the given
    (mu, 1/s) (genio.cpp:150-185). Returns the dense p x n fp64 matrix in
    column-major order (the layout DenseOperator's Eigen GEMV reads)."""
    d = bed_decode(payload, p, n)
    mean = marker_means(marker_counts(payload, p, n))
    X = np.empty((p, n), dtype=np.float64, order="F")
    step = max(1, (1 << 27) // max(n, 1))
    for j0 in range(0, p, step):  # row blocks: bounded temporaries
        j1 = min(p, j0 + step)
        blk = d[j0:j1].astype(np.float64)
        miss = d[j0:j1] == 3
        blk[miss] = np.broadcast_to(mean[j0:j1, None], blk.shape)[miss]
        X[j0:j1] = (blk - np.asarray(mu)[j0:j1, None]) * np.asarray(inv_s)[j0:j1, None]
    return X


class DenseOracle:
    def __init__(self, X):
        self.X = np.asfortranarray(np.asarray(X, dtype=np.float64))
        self.op = orc_op()
        _o.orc_dense_op(C.byref(self.op), self.X.ctypes.data_as(PD), self.X.shape[0],
                        self.X.shape[1])


def norm_estimate(o, iters=20, seed=0x9E3779B97F4A7C15):
    return _o.orc_norm_estimate(C.byref(o.op), iters, seed)


def adjoint_mismatch(o, seed=7):
    return _o.orc_adjoint_mismatch(C.byref(o.op), seed)


def cgs2(basis, v, coeffs=None):
    Q = np.asfortranarray(np.asarray(basis, dtype=np.float64))
    v = _f64(v).copy()
    cf = np.zeros(Q.shape[1]) if coeffs is None else coeffs
    na = _o.orc_cgs2(Q.ctypes.data_as(PD), Q.shape[0], Q.shape[1], _pd(v), _pd(cf))
    return na, v


def svd_small(M):
    M = np.asfortranarray(np.asarray(M, dtype=np.float64))
    r, c = M.shape
    k = min(r, c)
    U, s, V = np.empty(r * k), np.empty(k), np.empty(c * k)
    _o.orc_svd_small(M.ctypes.data_as(PD), r, c, _pd(U), _pd(s), _pd(V))
    return U.reshape(k, r).T, s, V.reshape(k, c).T


# ------------------------------------------------------------------ GKL
@dataclass
class Options:
    k: int = 10
    tol: float = 1e-8
    max_mvps: int = 1000000
    reorth: int = 1  # 0 full, 1 partial
    omega: float = 1e-8
    one_sided: bool = False
    restart: int = 0  # 0 none, 1 thick
    max_subspace: int = 40
    keep: int = 20
    seed: int = 0
    record_history: bool = False
    omega_recurrence: int = 1

    def c(self):
        return orc_gkl_options(int(self.k), float(self.tol), int(self.max_mvps), int(self.reorth),
                               float(self.omega), int(bool(self.one_sided)), int(self.restart),
                               int(self.max_subspace), int(self.keep),
                               int(self.seed) & 0xFFFFFFFFFFFFFFFF, int(bool(self.record_history)),
                               int(self.omega_recurrence))

    @staticmethod
    def from_gkl(o) -> "Options":
        return Options(k=o.k, tol=o.tol, max_mvps=o.max_mvps, reorth=int(o.reorth),
                       omega=o.omega, one_sided=o.one_sided, restart=int(o.restart),
                       max_subspace=o.max_subspace, keep=o.keep, seed=o.seed,
                       record_history=o.record_history,
                       omega_recurrence=int(getattr(o, "omega_recurrence", 1)))


def validate(opts: Options, m, n):
    msg = C.create_string_buffer(256)
    rc = _o.orc_gkl_options_validate(C.byref(opts.c()), m, n, msg, 256)
    if rc:
        raise ValueError(msg.value.decode())


@dataclass
class SvdlOut:
    singvals: np.ndarray
    U: np.ndarray
    V: np.ndarray
    err: np.ndarray
    converged: np.ndarray
    mvps: int
    steps: int
    restarts: int
    reorth_count: int
    deflations: int
    all_converged: bool
    wall_seconds: float
    ritz_history: list


def svdl(o, opts: Options) -> SvdlOut:
    res = orc_svdl_result()
    msg = C.create_string_buffer(256)
    oc = opts.c()
    rc = _o.orc_svdl(C.byref(o.op), C.byref(oc), C.byref(res), msg, 256)
    if rc:
        raise ValueError(msg.value.decode())
    try:
        cnt = res.count
        m, n = o.op.rows, o.op.cols

        def arr(p, k):
            return np.ctypeslib.as_array(p, shape=(k,)).copy() if k > 0 else np.zeros(0)
        hist = []
        if res.history_len > 0:
            h = arr(res.ritz_history, res.history_len * opts.k).reshape(res.history_len, opts.k)
            hist = [row[~np.isnan(row)] for row in h]
        return SvdlOut(
            singvals=arr(res.singvals, cnt),
            U=arr(res.U, m * cnt).reshape(cnt, m).T if cnt else np.zeros((m, 0)),
            V=arr(res.V, n * cnt).reshape(cnt, n).T if cnt else np.zeros((n, 0)),
            err=arr(res.err, cnt),
            converged=(np.ctypeslib.as_array(res.converged, shape=(cnt,)).astype(bool).copy()
                       if cnt else np.zeros(0, dtype=bool)),
            mvps=res.mvps, steps=res.steps, restarts=res.restarts,
            reorth_count=res.reorth_count, deflations=res.deflations,
            all_converged=bool(res.all_converged), wall_seconds=res.wall_seconds,
            ritz_history=hist)
    finally:
        _o.orc_svdl_result_free(C.byref(res))


class Lanczos:
    """LanczosFactorization + bidiag_step on the CPU (KAT tests)."""

    def __init__(self, o, capacity, start, rng_seed=1):
        self.o = o
        self.f = orc_lanczos()
        start = _f64(start)
        rc = _o.orc_lanczos_init(C.byref(self.f), o.op.rows, o.op.cols, capacity, _pd(start))
        if rc:
            raise ValueError(f"LanczosFactorization: init failed ({rc})")
        self.rng = orc_rng()
        _o.orc_rng_init(C.byref(self.rng), int(rng_seed))
        self.mvps = C.c_long(0)

    def __del__(self):
        try:
            _o.orc_lanczos_free(C.byref(self.f))
        except Exception:
            pass

    def step(self, opts: Options, norm_scale: float):
        info = orc_step_info()
        oc = opts.c()
        rc = _o.orc_bidiag_step(C.byref(self.o.op), C.byref(self.f), C.byref(oc),
                                C.byref(self.rng), float(norm_scale), C.byref(self.mvps),
                                C.byref(info))
        if rc:
            raise RuntimeError("bidiag_step: logic error")
        return info

    @property
    def steps(self):
        return self.f.j

    def left_basis(self):
        m, j = self.f.m, self.f.j
        return np.ctypeslib.as_array(self.f.U, shape=(m * self.f.cap,))[: m * j].reshape(j, m).T.copy()

    def right_basis(self):
        n, j = self.f.n, self.f.j
        return np.ctypeslib.as_array(self.f.V, shape=(n * (self.f.cap + 1),))[: n * (j + 1)].reshape(
            j + 1, n).T.copy()

    def projected(self):
        cap, j = self.f.cap, self.f.j
        B = np.ctypeslib.as_array(self.f.B, shape=(cap * cap,)).reshape(cap, cap).T
        return B[:j, :j].copy()

    def coupling(self):
        return np.ctypeslib.as_array(self.f.coupling, shape=(self.f.cap,))[: self.f.j].copy()

    def compress_exhausted(self):  # gkl.cpp:380-409
        _o.orc_compress_exhausted(C.byref(self.f))

    def deflate_right(self):  # gkl.cpp:178-204
        _o.orc_deflate_right(C.byref(self.f), C.byref(self.rng))

    @property
    def right_exhausted(self):
        return bool(self.f.right_exhausted)

    def error_metric_l1(self, tol, k):  # gkl.cpp:411-414
        r = orc_ritz()
        _o.orc_ritz_extract(C.byref(self.f), float(tol), C.byref(r))
        try:
            return _o.orc_error_metric_l1(C.byref(r), int(k))
        finally:
            _o.orc_ritz_free(C.byref(r))

    def ritz(self, tol):
        r = orc_ritz()
        _o.orc_ritz_extract(C.byref(self.f), float(tol), C.byref(r))
        j = r.j
        try:
            if j == 0:
                return np.zeros(0), np.zeros(0), np.zeros(0)
            return (np.ctypeslib.as_array(r.values, shape=(j,)).copy(),
                    np.ctypeslib.as_array(r.err_crude, shape=(j,)).copy(),
                    np.ctypeslib.as_array(r.converged, shape=(j,)).astype(bool).copy())
        finally:
            _o.orc_ritz_free(C.byref(r))

    def thick_restart(self, keep):
        if _o.orc_thick_restart(C.byref(self.f), keep):
            raise ValueError("thick_restart: need 1 <= keep < steps")


# ------------------------------------------------------------------ synth
def synth_bed(spec, j0: int = 0, j1: Optional[int] = None) -> np.ndarray:
    """CPU bytes of the counter-based generator for markers [j0, j1)."""
    j1 = spec.p if j1 is None else j1
    keep = []

    def ptr(a, ct):
        if a is None:
            return C.POINTER(ct)()
        a = np.ascontiguousarray(a)
        keep.append(a)
        return a.ctypes.data_as(C.POINTER(ct))
    s = orc_synth_spec(spec.p, spec.n, int(spec.seed), spec.npop,
                       ptr(np.asarray(spec.freq, dtype=np.float64), C.c_double),
                       ptr(None if spec.pop is None else np.asarray(spec.pop, dtype=np.int32),
                           C.c_int32),
                       ptr(None if spec.admix is None else np.asarray(spec.admix, np.float64),
                           C.c_double),
                       float(spec.missing_rate),
                       ptr(None if spec.copy_from is None else
                           np.asarray(spec.copy_from, dtype=np.int32), C.c_int32),
                       float(spec.copy_prob))
    out = np.empty((j1 - j0) * ((spec.n + 3) // 4), dtype=np.uint8)
    _o.orc_synth_bed(C.byref(s), j0, j1, out.ctypes.data_as(PU8))
    return out
