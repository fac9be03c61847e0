"""Host-side mirror of the reference's solver and operator API.

Python twin of ``gkpca::GklOptions``, ``svdl``, ``LinearOperator`` /
``DenseOperator`` and the ``LanczosFactorization`` step functions
(/root/reference/proj/include/gkpca/gkl.hpp:17-196, linop.hpp:13-64), bound
through the C ABI of libgkb.so. Same names, argument meaning and error
behaviour (ValueError for std::invalid_argument, LogicError for
std::logic_error), so the parity tests read like the reference's own tests.

Orientation follows the reference: an operator is m x n with
``apply(x) = X x`` and ``apply_adjoint(y) = X^T y``; a genotype operator is
markers x samples (m = p SNPs, n individuals).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

__all__ = [
    "ReorthMode", "RestartMode", "ScalingScheme", "GklOptions", "SvdlStats", "SvdlResult",
    "Context", "LinearOperator", "DenseOperator", "GenotypeOperator", "LanczosFactorization",
    "StepInfo", "StepStatus", "RitzSet", "svdl", "cgs2", "svd_small", "rng_uniform_symmetric",
    "partition_rows", "marker_scaling", "error_metric_l1", "pinned_empty", "bed_check", "rng_normal",
    "norm_estimate", "adjoint_mismatch",
]


def _pd(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a, n: Optional[int] = None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if n is not None and a.size != n:
        raise ValueError(f"length mismatch: expected {n}, got {a.size}")
    return a


def _out(out, n: int) -> np.ndarray:
    if out is None:
        return np.empty(n)
    if (not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.size != n
            or not out.flags.c_contiguous or not out.flags.writeable):
        raise ValueError(f"out must be a writeable contiguous float64 array of length {n}")
    return out


def bed_check(bed: str, bim: str, fam: str):
    """(p, n) of a PLINK fileset after read_bed's checks (genio.cpp:53-70);
    raises FormatError with the reference's messages. Needs no GPU."""
    p, n = C.c_int64(), C.c_int64()
    check(lib.gkb_bed_check(bed.encode(), bim.encode(), fam.encode(), C.byref(p), C.byref(n)))
    return p.value, n.value


def pinned_empty(n: int) -> np.ndarray:
    """Uninitialized float64 array of length n in page-locked host memory
    (gkb_host_alloc), freed when the array is garbage collected. Inputs and
    `out` arrays in pinned memory make gkb_op_apply's copies DMA-rate."""
    import weakref
    n = int(n)
    if n <= 0:
        raise ValueError("pinned_empty: n must be positive")
    ptr = C.c_void_p()
    check(lib.gkb_host_alloc(C.c_size_t(8 * n), C.byref(ptr)))
    buf = (C.c_double * n).from_address(ptr.value)
    arr = np.ctypeslib.as_array(buf)
    weakref.finalize(buf, lib.gkb_host_free, C.c_void_p(ptr.value))
    arr.setflags(write=True)
    return arr


class ReorthMode(enum.IntEnum):  # gkl.hpp:12
    kFull = 0
    kPartial = 1


class RestartMode(enum.IntEnum):  # gkl.hpp:13
    kNone = 0
    kThick = 1


class ScalingScheme(enum.IntEnum):  # genio.hpp:58-62 (+ BASELINE's hwe)
    kUnitVariance = 0
    kBinomial = 1
    kHwe = 2  # (g - 2f)/sqrt(2f(1-f)), BASELINE.json config standardization
    kNone = 3


class StepStatus(enum.IntEnum):  # gkl.hpp:111-116
    kOk = 0
    kBreakdownAlpha = 1
    kBreakdownBeta = 2


@dataclass
class GklOptions:
    """GklOptions (gkl.hpp:17-33): the reference's field names and defaults,
    plus one field the reference does not have: `omega_recurrence`. Its
    default 1 is NOT the reference's algorithm -- it adds the |coupling| nu
    term that the left recurrence of gkl.cpp:127-136 omits (the
    literal recurrence loses orthogonality on the config-2 model); 0 runs
    gkl.cpp:127-136 as written."""
    k: int = 10
    tol: float = 1e-8
    max_mvps: int = 1000000
    reorth: ReorthMode = ReorthMode.kPartial
    omega: float = 1e-8
    one_sided: bool = False
    restart: RestartMode = RestartMode.kNone
    max_subspace: int = 40
    keep: int = 20
    seed: int = 0
    record_history: bool = False
    # 1: complete left omega recurrence (default); 0: gkl.cpp:127-136 as written
    omega_recurrence: int = 1

    def _c(self) -> _lib.gkb_gkl_options:
        o = _lib.gkb_gkl_options()
        o.k = int(self.k)
        o.tol = float(self.tol)
        o.max_mvps = int(self.max_mvps)
        o.reorth = int(self.reorth)
        o.omega = float(self.omega)
        o.one_sided = int(bool(self.one_sided))
        o.restart = int(self.restart)
        o.max_subspace = int(self.max_subspace)
        o.keep = int(self.keep)
        o.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        o.record_history = int(bool(self.record_history))
        o.omega_recurrence = int(self.omega_recurrence)
        return o

    def validate(self, m: int, n: int) -> None:
        """GklOptions::validate (gkl.cpp:53-73): raises ValueError."""
        o = self._c()
        check(lib.gkb_gkl_options_validate(C.byref(o), int(m), int(n)))


@dataclass
class SvdlStats:  # gkl.hpp:170-180
    mvps: int = 0
    steps: int = 0
    restarts: int = 0
    reorth_count: int = 0
    deflations: int = 0
    converged: bool = False
    wall_seconds: float = 0.0
    ritz_history: List[np.ndarray] = field(default_factory=list)
    err_history: List[np.ndarray] = field(default_factory=list)
    device_seconds: float = 0.0
    host_syncs: int = 0
    fused_tails: int = 0  # right half-steps run as one fused launch (device path)


@dataclass
class SvdlResult:  # gkl.hpp:182-189
    singvals: np.ndarray
    U: np.ndarray
    V: np.ndarray
    err_estimates: np.ndarray
    converged: np.ndarray
    stats: SvdlStats


class Context:
    """Device context: shards + communicator (gkb_init / gkb_init_nccl)."""

    def __init__(self, devices: Sequence[int] = (0,), *, nccl: Optional[tuple] = None,
                 host_comm: Optional[tuple] = None):
        """devices: local shards (gkb_init). nccl=(device, unique_id, nranks,
        rank): one process per GPU over NCCL. host_comm=(device, nranks, rank,
        allreduce): SPMD with the sums done by `allreduce(a)`, which must
        replace the float64 numpy array `a` in place by its sum over all
        ranks (e.g. torch.distributed over gloo); it runs on a CUDA
        host-function thread and must not call into the library."""
        self._h = C.c_void_p()
        self._host_cb = None
        if host_comm is not None:
            device, nranks, rank, fn = host_comm

            def tramp(_user, buf, count, fn=fn):
                try:
                    fn(np.ctypeslib.as_array(buf, shape=(int(count),)))
                except BaseException as e:  # never unwind into the CUDA thread
                    import sys
                    import traceback
                    traceback.print_exc()
                    sys.stderr.flush()
                    os._exit(70)
            self._host_cb = _lib.HOST_ALLREDUCE_FN(tramp)
            check(lib.gkb_init_host_comm(int(device), int(nranks), int(rank), self._host_cb, None,
                                         C.byref(self._h)))
        elif nccl is not None:
            device, uid, nranks, rank = nccl
            buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
            check(lib.gkb_init_nccl(int(device), buf, int(nranks), int(rank), C.byref(self._h)))
        else:
            devs = (C.c_int * len(devices))(*devices)
            check(lib.gkb_init(len(devices), devs, C.byref(self._h)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib.gkb_nccl_unique_id(buf))
        return bytes(buf)

    def info(self):
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        check(lib.gkb_ctx_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def synchronize(self):
        check(lib.gkb_synchronize(self._h))

    def close(self):
        if self._h:
            check(lib.gkb_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context((0,))
    return _default_ctx


class LinearOperator:
    """LinearOperator (linop.hpp:13-39) backed by a device operator handle."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self._h = handle
        m, n = C.c_int64(), C.c_int64()
        check(lib.gkb_op_shape(self._h, C.byref(m), C.byref(n)))
        self._m, self._n = m.value, n.value

    def rows(self) -> int:
        return self._m

    def cols(self) -> int:
        return self._n

    @property
    def shape(self):
        return (self._m, self._n)

    def apply(self, x, out=None) -> np.ndarray:
        """y = X x (linop.hpp:20-22); raises ValueError on length mismatch.
        `out` (float64, length rows) receives the result; pass arrays from
        `pinned_empty` for DMA-rate host<->device copies."""
        x = _f64(x, self._n)
        y = _out(out, self._m)
        check(lib.gkb_op_apply(self._h, _pd(x), _pd(y)))
        return y

    def apply_adjoint(self, x, out=None) -> np.ndarray:
        """y = X^T x (linop.hpp:24-26); `out` as for apply (length cols)."""
        x = _f64(x, self._m)
        y = _out(out, self._n)
        check(lib.gkb_op_apply_adjoint(self._h, _pd(x), _pd(y)))
        return y

    def apply_block(self, X) -> np.ndarray:
        """Y = X_op X for a cols x k block (gkb_op_apply_block; k mvps)."""
        X = np.asfortranarray(np.asarray(X, dtype=np.float64))
        if X.ndim != 2 or X.shape[0] != self._n:
            raise ValueError(f"apply_block: expected a {self._n} x k block")
        k = X.shape[1]
        Y = np.empty((self._m, k), order="F")
        check(lib.gkb_op_apply_block(self._h, _pd(X), k, _pd(Y)))
        return Y

    def apply_adjoint_block(self, Y) -> np.ndarray:
        """Z = X_op^T Y for a rows x k block (gkb_op_apply_adjoint_block; k mvps)."""
        Y = np.asfortranarray(np.asarray(Y, dtype=np.float64))
        if Y.ndim != 2 or Y.shape[0] != self._m:
            raise ValueError(f"apply_adjoint_block: expected a {self._m} x k block")
        k = Y.shape[1]
        Z = np.empty((self._n, k), order="F")
        check(lib.gkb_op_apply_adjoint_block(self._h, _pd(Y), k, _pd(Z)))
        return Z

    def mvps(self) -> int:
        return int(lib.gkb_op_mvps(self._h))

    def bench(self, which: int, iters: int, flush_l2: bool = True):
        ms, main_ms, launches = C.c_double(), C.c_double(), C.c_int()
        check(lib.gkb_op_bench(self._h, int(which), int(iters), int(bool(flush_l2)), C.byref(ms),
                               C.byref(main_ms), C.byref(launches)))
        return ms.value, main_ms.value, launches.value

    def close(self):
        if self._h:
            check(lib.gkb_op_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DenseOperator(LinearOperator):
    """DenseOperator (linop.hpp:43-64) on the device (column-major copy)."""

    def __init__(self, X, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        X = np.asfortranarray(np.asarray(X, dtype=np.float64))
        if X.ndim != 2:
            raise ValueError("DenseOperator: 2-D matrix required")
        h = C.c_void_p()
        check(lib.gkb_dense_create(ctx._h, X.ctypes.data_as(C.POINTER(C.c_double)), X.shape[0],
                                   X.shape[1], C.byref(h)))
        super().__init__(ctx, h)


class GenotypeOperator(LinearOperator):
    """Packed 2-bit genotype operator in HBM (p markers x n samples).

    Entry (j, s) = (d_js - mu_j) * inv_s_j for an observed dosage, 0 for a
    missing one: impute_mean + standardize (genio.cpp:124-185) applied
    implicitly, never densified (load_matrix, gkpca.cpp:89-108, is replaced).
    """

    def __init__(self, ctx: Context, handle: C.c_void_p, p: int, n: int):
        super().__init__(ctx, handle)
        self.p, self.n = p, n

    @classmethod
    def from_bed_payload(cls, payload, p: int, n: int, ctx: Optional[Context] = None,
                         scheme: Optional[ScalingScheme] = ScalingScheme.kHwe):
        ctx = ctx or default_context()
        buf = np.ascontiguousarray(np.frombuffer(payload, dtype=np.uint8)
                                   if isinstance(payload, (bytes, bytearray, memoryview))
                                   else np.asarray(payload, dtype=np.uint8))
        stride = (n + 3) // 4
        if buf.size != p * stride:
            raise _lib.FormatError(
                f"payload size mismatch (expected {p * stride} bytes, found {buf.size})")
        h = C.c_void_p()
        check(lib.gkb_geno_from_bed(ctx._h, buf.ctypes.data_as(C.POINTER(C.c_uint8)), p, n,
                                    C.byref(h)))
        op = cls(ctx, h, p, n)
        if scheme is not None:
            op.standardize(scheme)
        return op

    @classmethod
    def from_bed_file(cls, bed: str, bim: Optional[str] = None, fam: Optional[str] = None,
                      ctx: Optional[Context] = None,
                      scheme: Optional[ScalingScheme] = ScalingScheme.kHwe):
        """Streams a PLINK .bed file into HBM (gkb_geno_from_bed_file; read_bed's
        checks, genio.cpp:53-70). `bed` may be the fileset prefix; .bim/.fam default
        to the same prefix."""
        from . import genio
        b, bi, fa = genio.bed_paths(bed)
        bim, fam = bim or bi, fam or fa
        p, n = bed_check(b, bim, fam)  # FormatError before touching the device
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib.gkb_geno_from_bed_file(ctx._h, b.encode(), bim.encode(), fam.encode(),
                                         C.byref(h)))
        op = cls(ctx, h, p, n)
        if scheme is not None:
            op.standardize(scheme)
        return op

    @classmethod
    def from_synth(cls, spec, ctx: Optional[Context] = None,
                   scheme: Optional[ScalingScheme] = ScalingScheme.kHwe):
        """Genotypes generated on the device (see synth.py)."""
        ctx = ctx or default_context()
        cs, keep = spec.to_c()
        h = C.c_void_p()
        check(lib.gkb_geno_from_synth(ctx._h, C.byref(cs), C.byref(h)))
        del keep
        op = cls(ctx, h, spec.p, spec.n)
        if scheme is not None:
            op.standardize(scheme)
        return op

    def counts(self) -> np.ndarray:
        """Per-marker [n0, n1, n2, nmissing] counted on the device."""
        out = np.zeros((self.p, 4), dtype=np.int64)
        check(lib.gkb_geno_counts(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def standardize(self, scheme: ScalingScheme) -> None:
        check(lib.gkb_geno_standardize(self._h, int(scheme)))

    def set_scaling(self, mu, inv_s) -> None:
        mu, inv_s = _f64(mu, self.p), _f64(inv_s, self.p)
        check(lib.gkb_geno_set_scaling(self._h, _pd(mu), _pd(inv_s)))

    def marker_scan(self, y, Z=None, unbiased: bool = False):
        """Per-marker fits y ~ [1, m_i, Z] on the device (gkb_geno_marker_scan):
        (beta, se, intercept, sigma2, dependent) arrays of length p."""
        y = _f64(y, self.n)
        Zm = np.zeros((self.n, 0)) if Z is None else np.asfortranarray(
            np.asarray(Z, dtype=np.float64).reshape(self.n, -1))
        k = Zm.shape[1]
        outs = [np.empty(self.p) for _ in range(4)]
        dep = np.empty(self.p, dtype=np.int32)
        zp = _pd(Zm) if k else C.POINTER(C.c_double)()
        check(lib.gkb_geno_marker_scan(self._h, _pd(y), zp, k, int(bool(unbiased)),
                                       *[_pd(o) for o in outs],
                                       dep.ctypes.data_as(C.POINTER(C.c_int32))))
        return (*outs, dep.astype(bool))

    def scaling(self):
        mu, inv_s = np.empty(self.p), np.empty(self.p)
        check(lib.gkb_geno_get_scaling(self._h, _pd(mu), _pd(inv_s)))
        return mu, inv_s

    def read_bed(self, row0: int = 0, nrows: Optional[int] = None) -> np.ndarray:
        nrows = self.p - row0 if nrows is None else nrows
        out = np.empty(nrows * ((self.n + 3) // 4), dtype=np.uint8)
        check(lib.gkb_geno_read_bed(self._h, row0, nrows, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out

    def modes(self):
        """(layouts, dense_missing): 2 = both tile layouts, 1 = single-layout
        mode; dense_missing = indicator MMAs instead of per-CTA lists."""
        a, b = C.c_int(), C.c_int()
        check(lib.gkb_geno_layouts(self._h, C.byref(a), C.byref(b)))
        return a.value, bool(b.value)

    def info(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.gkb_geno_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"nmissing": a.value, "packed_bytes": b.value, "device_bytes": c.value}


class _OwnedArray(np.ndarray):
    """A view of library-owned memory; `_owner` frees it with the last view."""


class _SvdlResultOwner:
    def __init__(self, res):
        self.res = res

    def __del__(self):
        try:
            check(lib.gkb_svdl_result_free(self.res))
        except Exception:
            pass


def svdl(op: LinearOperator, opts: GklOptions) -> SvdlResult:
    """svdl (gkl.hpp:196, gkl.cpp:416-514). U and V are Fortran-ordered views
    of the library's result buffers (no copy); the buffers are released with
    the last view."""
    o = opts._c()
    res = C.POINTER(_lib.gkb_svdl_result)()
    check(lib.gkb_svdl(op._h, C.byref(o), C.byref(res)))
    owner = _SvdlResultOwner(res)
    r = res.contents
    cnt, m, n = r.count, r.m, r.n

    def arr(p, k):
        return np.ctypeslib.as_array(p, shape=(k,)).copy() if k > 0 else np.zeros(0)

    def cols(p, rows):  # column-major rows x cnt, viewed in place
        if not cnt:
            return np.zeros((rows, 0))
        v = np.ctypeslib.as_array(p, shape=(cnt, rows)).T.view(_OwnedArray)
        v._owner = owner
        return v

    singvals = arr(r.singvals, cnt)
    U = cols(r.U, m)
    V = cols(r.V, n)
    err = arr(r.err_estimates, cnt)
    conv = (np.ctypeslib.as_array(r.converged, shape=(cnt,)).astype(bool).copy()
            if cnt else np.zeros(0, dtype=bool))
    st = SvdlStats(mvps=r.mvps, steps=r.steps, restarts=r.restarts,
                   reorth_count=r.reorth_count, deflations=r.deflations,
                   converged=bool(r.all_converged), wall_seconds=r.wall_seconds,
                   device_seconds=r.device_seconds, host_syncs=r.host_syncs,
                   fused_tails=r.fused_tails)
    if r.history_len > 0:
        k = int(opts.k)
        h = arr(r.ritz_history, r.history_len * k).reshape(r.history_len, k)
        e = arr(r.err_history, r.history_len * k).reshape(r.history_len, k)
        st.ritz_history = [row[~np.isnan(row)] for row in h]
        st.err_history = [row[~np.isnan(row)] for row in e]
    return SvdlResult(singvals, U, V, err, conv, st)


@dataclass
class StepInfo:  # gkl.hpp:118-125
    status: StepStatus
    reorthogonalized_left: bool
    reorthogonalized_right: bool
    alpha: float
    beta: float


@dataclass
class RitzSet:  # gkl.hpp:39-46
    values: np.ndarray
    left_coeffs: np.ndarray
    right_coeffs: np.ndarray
    err_estimates: np.ndarray
    err_crude: np.ndarray
    converged: np.ndarray


class LanczosFactorization:
    """LanczosFactorization (gkl.hpp:59-109) with device-resident bases.

    The Rng used for deflation vectors is owned here (seed ``rng_seed``),
    standing in for the ``Rng&`` argument of bidiag_step.
    """

    def __init__(self, op: LinearOperator, capacity: int, start, rng_seed: int = 1):
        start = _f64(start, op.cols())
        self.op = op
        self._h = C.c_void_p()
        check(lib.gkb_lanczos_create(op._h, int(capacity), _pd(start), int(rng_seed),
                                     C.byref(self._h)))

    def _info(self):
        s, c, r = C.c_int64(), C.c_int64(), C.c_int()
        check(lib.gkb_lanczos_info(self._h, C.byref(s), C.byref(c), C.byref(r)))
        return s.value, c.value, bool(r.value)

    def rows(self):
        return self.op.rows()

    def cols(self):
        return self.op.cols()

    def steps(self) -> int:
        return self._info()[0]

    def capacity(self) -> int:
        return self._info()[1]

    def right_exhausted(self) -> bool:
        return self._info()[2]

    def _get(self):
        j = self.steps()
        m, n = self.rows(), self.cols()
        U = np.empty(m * j)
        V = np.empty(n * (j + 1))
        B = np.empty(j * j)
        cp = np.empty(j)
        ol = np.empty(j)
        orr = np.empty(j + 1)
        check(lib.gkb_lanczos_get(self._h, _pd(U), _pd(V), _pd(B), _pd(cp), _pd(ol), _pd(orr)))
        return (U.reshape(j, m).T, V.reshape(j + 1, n).T, B.reshape(j, j).T, cp, ol, orr)

    def left_basis(self):
        return self._get()[0]

    def right_basis(self):
        return self._get()[1]

    def projected(self):
        return self._get()[2]

    def residual_coupling(self):
        return self._get()[3]

    def omega_left(self):
        return self._get()[4]

    def omega_right(self):
        return self._get()[5]

    def alphas(self):
        return np.diag(self.projected()).copy()

    def betas(self):  # gkl.cpp:100-106
        B = self.projected()
        j = B.shape[0]
        out = np.empty(j)
        for i in range(j - 1):
            out[i] = B[i, i + 1]
        if j:
            out[j - 1] = np.linalg.norm(self.residual_coupling())
        return out

    def bidiag_step(self, opts: GklOptions, norm_scale: float) -> StepInfo:
        o = opts._c()
        st, rl, rr = C.c_int(), C.c_int(), C.c_int()
        a, b = C.c_double(), C.c_double()
        check(lib.gkb_bidiag_step(self._h, C.byref(o), float(norm_scale), C.byref(st),
                                  C.byref(rl), C.byref(rr), C.byref(a), C.byref(b)))
        return StepInfo(StepStatus(st.value), bool(rl.value), bool(rr.value), a.value, b.value)

    def ritz_extract(self, tol: float) -> RitzSet:
        j = self.steps()
        vals, wl, wr = np.empty(j), np.empty(j * j), np.empty(j * j)
        err, crude = np.empty(j), np.empty(j)
        conv = np.empty(j, dtype=np.int32)
        check(lib.gkb_ritz_extract(self._h, float(tol), _pd(vals), _pd(wl), _pd(wr), _pd(err),
                                   _pd(crude), conv.ctypes.data_as(C.POINTER(C.c_int32))))
        return RitzSet(vals, wl.reshape(j, j).T, wr.reshape(j, j).T, err, crude, conv.astype(bool))

    def thick_restart(self, keep: int) -> None:
        check(lib.gkb_thick_restart(self._h, int(keep)))

    def compress_exhausted(self) -> None:
        check(lib.gkb_compress_exhausted(self._h))

    def deflate_right(self) -> None:  # gkl.cpp:178-204 (draws from this factorization's Rng)
        check(lib.gkb_deflate_right(self._h))

    def close(self):
        if self._h:
            check(lib.gkb_lanczos_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def geno_plan(p_loc: int, n: int, missing_fraction: float, free_bytes: int):
    """Layout plan of one shard (gkb_geno_plan): (layouts, dual_bytes, single_bytes)."""
    a, b, c = C.c_int(), C.c_int64(), C.c_int64()
    check(lib.gkb_geno_plan(int(p_loc), int(n), float(missing_fraction), int(free_bytes),
                            C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def error_metric_l1(ritz: RitzSet, k: int) -> float:  # gkl.cpp:411-414
    return float(np.sum(ritz.err_crude[: min(k, ritz.err_crude.size)]))


def cgs2(basis, v, coeffs=None, ctx: Optional[Context] = None):
    """cgs2 (orth.hpp:19-44) on the device; returns (norm_after, v)."""
    ctx = ctx or default_context()
    Q = np.asfortranarray(np.asarray(basis, dtype=np.float64))
    v = _f64(v).copy()
    if Q.ndim != 2 or Q.shape[0] != v.size:
        raise ValueError("cgs2: basis rows must match the vector length")
    cf = np.zeros(Q.shape[1]) if coeffs is None else _f64(coeffs, Q.shape[1])
    na = C.c_double()
    check(lib.gkb_cgs2(ctx._h, Q.ctypes.data_as(C.POINTER(C.c_double)), Q.shape[0], Q.shape[1],
                       _pd(v), _pd(cf), C.byref(na)))
    if coeffs is not None:
        coeffs[...] = cf
    return na.value, v


def svd_small(M):
    """svd_small (small_svd.cpp:14-28): (U, s, V) with s descending."""
    M = np.asfortranarray(np.asarray(M, dtype=np.float64))
    r, c = M.shape
    k = min(r, c)
    U, s, V = np.empty(r * k), np.empty(k), np.empty(c * k)
    check(lib.gkb_svd_small(M.ctypes.data_as(C.POINTER(C.c_double)), r, c, _pd(U), _pd(s), _pd(V)))
    return U.reshape(k, r).T, s, V.reshape(k, c).T


def rng_uniform_symmetric(seed: int, n: int) -> np.ndarray:
    """Rng(seed).uniform_symmetric() x n (rng.hpp:27; gkl.cpp:428-429)."""
    out = np.empty(n)
    check(lib.gkb_rng_fill_symmetric(int(seed) & 0xFFFFFFFFFFFFFFFF, n, _pd(out)))
    return out


def norm_estimate(op: LinearOperator, iters: int = 20, seed: int = 0x9E3779B97F4A7C15) -> float:
    """norm_estimate (linop.hpp:122-123, linop.cpp:9-28): ||X z|| after `iters`
    power iterations on X^T X from a seeded uniform start -- a lower estimate of
    sigma_1. 2 iters + 1 products on the device operator."""
    n = op.cols()
    if n == 0 or op.rows() == 0:
        return 0.0
    z = rng_uniform_symmetric(seed, n)
    zn = float(np.linalg.norm(z))
    if zn == 0.0:
        z[0] = zn = 1.0
    z = z / zn
    for _ in range(int(iters)):
        w = op.apply_adjoint(op.apply(z))
        wn = float(np.linalg.norm(w))
        if wn == 0.0:  # z reached the null space exactly
            return 0.0
        z = w / wn
    return float(np.linalg.norm(op.apply(z)))


def adjoint_mismatch(op: LinearOperator, seed: int = 7) -> float:
    """adjoint_mismatch (linop.hpp:125-127, linop.cpp:30-39): |u'(X v) - (X^T u)'v|
    / (||u|| ||v||) on normal probes v (cols) then u (rows) from one stream."""
    n, m = op.cols(), op.rows()
    r = rng_normal(seed, n + m)
    v, u = r[:n], r[n:]
    left = float(u @ op.apply(v))
    right = float(op.apply_adjoint(u) @ v)
    scale = float(np.linalg.norm(u) * np.linalg.norm(v))
    return 0.0 if scale == 0.0 else abs(left - right) / scale


def rng_normal(seed: int, n: int) -> np.ndarray:
    """Rng(seed).normal() x n (Box-Muller, rng.hpp:46-60)."""
    out = np.empty(n)
    check(lib.gkb_rng_fill_normal(int(seed) & 0xFFFFFFFFFFFFFFFF, n, _pd(out)))
    return out


def partition_rows(m: int, nparts: int) -> np.ndarray:
    out = np.empty(nparts + 1, dtype=np.int64)
    check(lib.gkb_partition_rows(int(m), int(nparts), out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def marker_scaling(counts, n: int, scheme: ScalingScheme):
    counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int64).reshape(-1, 4))
    p = counts.shape[0]
    mu, inv_s = np.empty(p), np.empty(p)
    check(lib.gkb_marker_scaling(counts.ctypes.data_as(C.POINTER(C.c_int64)), p, int(n),
                                 int(scheme), _pd(mu), _pd(inv_s)))
    return mu, inv_s
