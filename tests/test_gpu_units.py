"""Unit parity of the device primitives against the reference's known answers
and the CPU oracle (through the C ABI):

* cgs2 on the device (gkb_cgs2) on the reference's KATs
  (/root/reference/proj/tests/test_linops.cpp:120-178) and GPU vs oracle on
  random bases, including a basis wider than the old fixed result buffer;
* the breakdown paths -- compress_exhausted (gkl.cpp:380-409) and
  deflate_right (gkl.cpp:178-204), both its random-vector branch and its
  exhausted branch -- step by step, GPU factorization vs oracle factorization
  on the same operator, start vector and Rng seed;
* error_metric_l1 (gkl.cpp:411-414).
"""
import numpy as np
import pytest

from conftest import principal_angles, rel_err, sigma_rel_err

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- cgs2
def test_cgs2_reference_kats(gkb, orc):  # test_linops.cpp:120-178
    Q = np.zeros((4, 1))
    Q[0, 0] = 1.0
    na, v = gkb.cgs2(Q, [0, 1.0, 0, 0])  # already orthogonal
    assert abs(na - 1.0) <= 1e-15 and abs(v[0]) <= 1e-15 and abs(v[1] - 1.0) <= 1e-15
    na, v = gkb.cgs2(Q, [1.0, 0, 0, 0])  # inside the span
    assert na <= 1e-14
    v0 = np.array([1.0, 1e-9, 0, 0])  # near-parallel: second pass
    na, v = gkb.cgs2(Q, v0)
    assert abs(na - 1e-9) <= 1e-12 * 1e-9
    assert abs(Q[:, 0] @ v) <= 1e-12 * np.linalg.norm(v0)
    g = orc.gaussian_matrix(5, 1, 3)[:, 0]  # empty basis: identity
    na, v = gkb.cgs2(np.zeros((5, 0)), g)
    assert abs(na - np.linalg.norm(g)) <= 1e-15 * na and np.array_equal(v, g)


def test_cgs2_coefficient_recovery_vs_oracle(gkb, orc):  # test_linops.cpp:153-169
    Qf = np.linalg.qr(orc.gaussian_matrix(50, 10, 77))[0]
    r = orc.Rng(78)
    for _ in range(20):
        v0 = np.array([r.uniform_symmetric() for _ in range(50)])
        cf = np.zeros(10)
        na, v = gkb.cgs2(Qf, v0, cf)
        assert np.abs(Qf.T @ v).max() <= 1e-12 * np.linalg.norm(v0)
        assert abs(na - np.linalg.norm(v)) <= 1e-13 * na
        assert np.abs(v0 - Qf @ cf - v).max() <= 1e-13 * np.linalg.norm(v0)
        cfo = np.zeros(10)
        nao, vo = orc.cgs2(Qf, v0, cfo)
        assert abs(na - nao) <= 1e-13 * nao
        assert rel_err(v, vo) <= 1e-12 and rel_err(cf, cfo) <= 1e-12


@pytest.mark.parametrize("length,ncols", [(100_000, 40), (4096, 300), (20_000, 61)])
def test_cgs2_tall_bases_vs_oracle(gkb, orc, length, ncols):
    """The basis shapes of the solver (len up to n, j up to cap + 1)."""
    rng = np.random.default_rng(length + ncols)
    Q = np.linalg.qr(rng.standard_normal((length, ncols)))[0]
    for t in range(3):
        v0 = rng.standard_normal(length)
        if t == 1:  # nearly inside the span: the second pass runs
            v0 = Q @ rng.standard_normal(ncols) + 1e-9 * v0
        cf, cfo = np.zeros(ncols), np.zeros(ncols)
        na, v = gkb.cgs2(Q, v0, cf)
        nao, vo = orc.cgs2(Q, v0, cfo)
        # cancellation: the residual of a nearly-in-span vector carries
        # eps * |v0| absolute error (the reference's bound, test_linops.cpp:161-167)
        assert abs(na - nao) <= 1e-13 * np.linalg.norm(v0)
        assert np.abs(v - vo).max() <= 1e-13 * np.abs(v0).max()
        assert rel_err(cf, cfo) <= 1e-12
        assert np.abs(Q.T @ v).max() <= 1e-12 * np.linalg.norm(v0)


def test_cgs2_basis_wider_than_old_result_buffer(gkb):
    """2 ncols + 5 result slots with ncols > 32766 (the result buffers grow
    with the basis; they were a fixed 65,536 doubles)."""
    ncols, length = 40_000, 100
    Q = np.zeros((length, ncols))
    Q[0, 0] = 1.0  # a valid (zero-padded) basis: only e1 carries weight
    v0 = np.zeros(length)
    v0[0], v0[1] = 1.0, 1e-9  # near-parallel: the second pass runs
    cf = np.zeros(ncols)
    na, v = gkb.cgs2(Q, v0, cf)
    assert abs(na - 1e-9) <= 1e-12 * 1e-9
    assert abs(cf[0] - 1.0) <= 1e-15 and np.all(cf[1:] == 0.0)
    assert abs(v[0]) <= 1e-18 and abs(v[1] - 1e-9) <= 1e-21


# ---------------------------------------------------------------- breakdown paths
def _block_diag(m1, n1, m2, n2, seed):
    rng = np.random.default_rng(seed)
    X = np.zeros((m1 + m2, n1 + n2))
    X[:m1, :n1] = rng.standard_normal((m1, n1))
    X[m1:, n1:] = rng.standard_normal((m2, n2))
    return X


def _cases():
    rng = np.random.default_rng(11)
    out = []
    for (m, n, r) in [(60, 40, 3), (40, 60, 5), (50, 50, 1)]:
        X = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
        out.append(("lowrank%dx%dr%d" % (m, n, r), X, None))
    # right Krylov space closes after 10 steps with j < n: beta breakdown and
    # deflate_right's random-vector branch inside bidiag_step
    X = _block_diag(15, 10, 15, 10, 5)
    s = np.zeros(20)
    s[:10] = np.random.default_rng(6).standard_normal(10)
    out.append(("blockdiag", X, s))
    out.append(("tall30x8", rng.standard_normal((30, 8)), None))  # beta breakdown at j = n
    return out


@pytest.mark.parametrize("name,X,start", _cases(), ids=[c[0] for c in _cases()])
@pytest.mark.parametrize("reorth", [0, 1])
def test_breakdown_paths_vs_oracle(gkb, orc, name, X, start, reorth):
    m, n = X.shape
    if start is None:
        r = orc.Rng(5)
        start = np.array([r.uniform_symmetric() for _ in range(n)])
    cap = min(20, m, n)
    g = gkb.LanczosFactorization(gkb.DenseOperator(X), cap, start, rng_seed=9)
    o = orc.Lanczos(orc.DenseOracle(X), cap, start, rng_seed=9)
    gopts = gkb.GklOptions(k=3, reorth=gkb.ReorthMode(reorth), tol=1e-10)
    oopts = orc.Options.from_gkl(gopts)
    ns_g = ns_o = 0.0
    seen = set()
    for _ in range(40):
        if g.steps() >= min(m, n) or g.right_exhausted():
            break
        ig = g.bidiag_step(gopts, ns_g)
        io = o.step(oopts, ns_o)
        assert int(ig.status) == io.status
        assert g.steps() == o.steps
        seen.add(int(ig.status))
        scale = max(1.0, abs(io.alpha))
        assert abs(ig.alpha - io.alpha) <= 1e-10 * scale
        assert abs(ig.beta - io.beta) <= 1e-10 * max(1.0, abs(io.beta))
        ns_g = max(ns_g, float(np.hypot(ig.alpha, ig.beta)))
        ns_o = max(ns_o, float(np.hypot(io.alpha, io.beta)))
        if int(ig.status) == 1:  # svdl's alpha-breakdown path (gkl.cpp:461-469)
            g.compress_exhausted()
            o.compress_exhausted()
            j = g.steps()
            assert sigma_rel_err(np.diag(g.projected()), np.diag(o.projected())) <= 1e-10
            if j:
                assert principal_angles(g.left_basis(), o.left_basis()) < 1e-7
            assert g.right_exhausted() and o.right_exhausted
            g.deflate_right()
            o.deflate_right()
            seen.add("deflate")
        assert g.right_exhausted() == o.right_exhausted
        Vg, Vo = g.right_basis(), o.right_basis()
        j = g.steps()
        # the pending right vector (deflation draws are bit-identical Rng
        # output; its cgs2 against V is sign-invariant)
        assert rel_err(Vg[:, j], Vo[:, j]) <= 1e-9 or (
            np.all(Vg[:, j] == 0) and np.all(Vo[:, j] == 0))
        if j:
            assert principal_angles(Vg[:, :j], Vo[:, :j]) < 1e-7
    assert seen - {0}, f"{name}: no breakdown reached"


def test_svdl_breakdowns_vs_oracle(gkb, orc):
    """Whole solves through the breakdown paths: deflation counts, mvps and
    singular values as the oracle's svdl."""
    for name, X, _ in _cases():
        for reorth in (0, 1):
            opts = gkb.GklOptions(k=3, reorth=gkb.ReorthMode(reorth), tol=1e-10, max_mvps=400,
                                  restart=gkb.RestartMode.kThick, max_subspace=min(20, *X.shape),
                                  keep=min(6, min(X.shape) - 1), seed=3)
            if opts.keep <= opts.k:
                opts.restart = gkb.RestartMode.kNone
            a = gkb.svdl(gkb.DenseOperator(X), opts)
            b = orc.svdl(orc.DenseOracle(X), orc.Options.from_gkl(opts))
            assert a.stats.deflations == b.deflations, name
            assert a.stats.mvps == b.mvps, name
            assert a.stats.restarts == b.restarts, name
            assert a.singvals.size == b.singvals.size
            s = np.linalg.svd(X, compute_uv=False)[: a.singvals.size]
            nz = s > 1e-8 * s[0]
            assert sigma_rel_err(a.singvals[nz], b.singvals[nz]) <= 1e-9, name


# ---------------------------------------------------------------- error_metric_l1
def test_error_metric_l1_vs_oracle(gkb, orc):  # gkl.cpp:411-414
    X = orc.gaussian_matrix(80, 50, 21)
    r = orc.Rng(4)
    start = np.array([r.uniform_symmetric() for _ in range(50)])
    g = gkb.LanczosFactorization(gkb.DenseOperator(X), 30, start, rng_seed=1)
    o = orc.Lanczos(orc.DenseOracle(X), 30, start, rng_seed=1)
    gopts = gkb.GklOptions(k=5, reorth=gkb.ReorthMode.kFull, tol=1e-8)
    oopts = orc.Options.from_gkl(gopts)
    ns_g = ns_o = 0.0
    for _ in range(12):
        ig, io = g.bidiag_step(gopts, ns_g), o.step(oopts, ns_o)
        ns_g = max(ns_g, float(np.hypot(ig.alpha, ig.beta)))
        ns_o = max(ns_o, float(np.hypot(io.alpha, io.beta)))
    rz = g.ritz_extract(1e-8)
    for k in (1, 5, 12, 40):
        e = gkb.error_metric_l1(rz, k)
        assert e == pytest.approx(float(np.sum(rz.err_crude[:min(k, rz.err_crude.size)])),
                                  rel=0, abs=0)
        assert e == pytest.approx(o.error_metric_l1(1e-8, k), rel=1e-9)
