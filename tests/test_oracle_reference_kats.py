"""Pins the CPU oracle on the reference's own known-answer and property tests
(the reference cannot be compiled here: Eigen3 and vendor/ are absent).

Sources: proj/tests/test_linops.cpp, test_gkl.cpp, test_genio.cpp and
acceptance.cpp criteria 1-2 (all under /root/reference). Independent dense
oracles are numpy/LAPACK.
"""
import numpy as np
import pytest

import oracle as O

EPS = np.finfo(float).eps


# ------------------------------------------------------------ Rng (rng.hpp)
def test_mt19937_64_engine_known_answer():
    r = O.Rng(5489)  # std::mt19937_64 default seed: 10000th output is fixed by the standard
    for _ in range(9999):
        r.bits()
    assert r.bits() == 9981545732273789042


def test_rng_semantics():  # test_linops.cpp:319-346
    r = O.Rng(42)
    for _ in range(1000):
        u = r.uniform()
        assert 0.0 <= u < 1.0
        s = r.uniform_symmetric()
        assert -1.0 <= s < 1.0
        k = r.uniform_int(3, 7)
        assert 3 <= k <= 7
    a, b = O.Rng(7), O.Rng(7)
    assert all(a.bits() == b.bits() for _ in range(100))
    c = O.Rng(9)
    xs = np.array([c.normal() for _ in range(200000)])
    assert abs(xs.mean()) <= 0.01 and abs((xs ** 2).mean() - 1.0) <= 0.02


def test_uniform_is_top53_bits():  # rng.hpp:24
    a, b = O.Rng(123), O.Rng(123)
    for _ in range(50):
        assert a.uniform() == (b.bits() >> 11) * 2.0 ** -53


# ------------------------------------------------------------ linops / orth
def test_dense_op_vs_naive_and_adjoint():  # test_linops.cpp:59-89
    for seed in (1, 2, 3):
        X = O.gaussian_matrix(17, 9, seed)
        d = O.DenseOracle(X)
        scale = O.norm_estimate(d, 20)
        assert O.adjoint_mismatch(d) <= 1e-10 * max(scale, 1.0)


def test_norm_estimate():  # test_linops.cpp:290-317
    d = O.DenseOracle(np.diag([5.0, 1.0]))
    est = O.norm_estimate(d, 30)
    assert abs(est - 5.0) <= 0.5 and est <= 5.0 * (1 + 1e-12)
    assert abs(O.norm_estimate(O.DenseOracle(np.eye(4)), 1) - 1.0) <= 1e-14
    assert O.norm_estimate(O.DenseOracle(np.zeros((3, 4))), 5) == 0.0
    for seed in range(1, 11):
        X = O.gaussian_matrix(30, 21, seed)
        est = O.norm_estimate(O.DenseOracle(X), 20)
        s1 = np.linalg.svd(X, compute_uv=False)[0]
        assert est <= s1 * (1 + 1e-12) and est >= 0.9 * s1


def test_cgs2_kats():  # test_linops.cpp:120-178
    Q = np.zeros((4, 1))
    Q[0, 0] = 1.0
    na, v = O.cgs2(Q, [0, 1.0, 0, 0])
    assert abs(na - 1.0) <= 1e-15 and abs(v[0]) <= 1e-15 and abs(v[1] - 1.0) <= 1e-15
    na, v = O.cgs2(Q, [1.0, 0, 0, 0])
    assert na <= 1e-14
    v0 = np.array([1.0, 1e-9, 0, 0])
    na, v = O.cgs2(Q, v0)
    assert abs(na - 1e-9) <= 1e-12 * 1e-9 and abs(Q[:, 0] @ v) <= 1e-12 * np.linalg.norm(v0)
    na, v = O.cgs2(np.zeros((5, 0)), O.gaussian_matrix(5, 1, 3)[:, 0])
    assert abs(na - np.linalg.norm(O.gaussian_matrix(5, 1, 3)[:, 0])) <= 1e-15 * na


def test_cgs2_coefficient_recovery():  # test_linops.cpp:153-169
    Qf = np.linalg.qr(O.gaussian_matrix(50, 10, 77))[0]
    r = O.Rng(78)
    for _ in range(20):
        v0 = np.array([r.uniform_symmetric() for _ in range(50)])
        cf = np.zeros(10)
        na, v = O.cgs2(Qf, v0, cf)
        assert np.abs(Qf.T @ v).max() <= 1e-12 * np.linalg.norm(v0)
        assert abs(na - np.linalg.norm(v)) <= 1e-13 * na
        assert np.abs(v0 - Qf @ cf - v).max() <= 1e-13 * np.linalg.norm(v0)


def test_svd_small():  # test_linops.cpp:230-288
    U, s, V = O.svd_small(np.diag([1.0, 3.0, 2.0]))
    assert np.allclose(s, [3, 2, 1], rtol=1e-15)
    U, s, V = O.svd_small(np.array([[0, 1.0], [1.0, 0]]))
    assert np.allclose(s, [1, 1], rtol=1e-15)
    r = O.Rng(1234)
    B = np.zeros((10, 10))
    for i in range(10):
        B[i, i] = 1.0 + r.uniform()
        if i + 1 < 10:
            B[i, i + 1] = r.uniform()
    ref = np.sqrt(np.maximum(0, np.linalg.eigvalsh(B.T @ B)[::-1]))
    assert np.allclose(O.svd_small(B)[1], ref, rtol=1e-10)
    for m, n in [(20, 7), (80, 100), (7, 20)]:
        M = O.gaussian_matrix(m, n, 900 + m)
        U, s, V = O.svd_small(M)
        k = min(m, n)
        assert np.abs(U.T @ U - np.eye(k)).max() <= 1e-12
        assert np.abs(V.T @ V - np.eye(k)).max() <= 1e-12
        assert np.abs(U @ np.diag(s) @ V.T - M).max() <= 1e-12 * s[0]
        assert np.all(np.diff(s) <= 0)
        assert np.allclose(s, np.linalg.svd(M, compute_uv=False), rtol=0, atol=1e-10 * s[0])
    M = O.gaussian_matrix(50, 3, 41) @ O.gaussian_matrix(40, 3, 42).T
    s = O.svd_small(M)[1]
    assert np.all(s[3:] <= 1e-12 * s[0])


# ------------------------------------------------------------ GKL (test_gkl.cpp)
def full():
    return O.Options(reorth=0)


def ident_defect(X, lz):
    U, Vf, B, cp = lz.left_basis(), lz.right_basis(), lz.projected(), lz.coupling()
    j = B.shape[0]
    return max(np.abs(X @ Vf[:, :j] - U @ B).max(),
               np.abs(X.T @ U - Vf[:, :j] @ B.T - np.outer(Vf[:, j], cp)).max())


def test_kat_single_step_diag():  # :53-65
    lz = O.Lanczos(O.DenseOracle(np.diag([2.0, 1.0])), 2, [1, 1.0])
    info = lz.step(full(), 0.0)
    assert info.status == 0 and abs(info.alpha - np.sqrt(2.5)) <= 1e-14 * np.sqrt(2.5)


def test_kat_one_by_one():  # :67-83
    lz = O.Lanczos(O.DenseOracle(np.array([[3.0]])), 1, [1.0])
    info = lz.step(full(), 3.0)
    assert info.status == 2 and abs(info.alpha - 3) <= 3e-15 and lz.f.right_exhausted
    with pytest.raises(RuntimeError):
        lz.step(full(), 3.0)


def test_kat_ritz_one_step():  # :85-103
    lz = O.Lanczos(O.DenseOracle(np.array([[3, 0.5], [0, 1.0]])), 2, [1.0, 0])
    info = lz.step(full(), 3.0)
    assert abs(info.alpha - 3) <= 3e-15 and abs(info.beta - 0.5) <= 1e-15
    vals, crude, conv = lz.ritz(1e-8)
    assert abs(vals[0] - 3) <= 3e-15 and abs(crude[0] - 0.5) <= 1e-15 and not conv[0]


def test_full_reorth_identities():  # :105-122
    X = O.gaussian_matrix(20, 30, 404)
    scale = np.linalg.svd(X, compute_uv=False)[0]
    lz = O.Lanczos(O.DenseOracle(X), 20, O.gaussian_matrix(30, 1, 405)[:, 0], 2)
    for _ in range(10):
        assert lz.step(full(), scale).status == 0
        assert ident_defect(X, lz) <= 1e-10 * scale
        U, V = lz.left_basis(), lz.right_basis()
        assert np.abs(U.T @ U - np.eye(U.shape[1])).max() <= 1e-12
        assert np.abs(V.T @ V - np.eye(V.shape[1])).max() <= 1e-12


def _decaying_case():
    m, n = 50, 60
    r = min(m, n)
    spec = 10.0 ** (-4.0 * np.arange(r) / (r - 1.0))
    QU = np.linalg.qr(O.gaussian_matrix(m, r, 7070))[0]
    QV = np.linalg.qr(O.gaussian_matrix(n, r, 7071))[0]
    return QU @ np.diag(spec) @ QV.T, spec, n


def _run_partial(recurrence):
    X, spec, n = _decaying_case()
    # The reference test starts from gaussian_matrix(n, 1, 7071), which is the
    # first column of the Gaussian draw behind QV (matrix_with_spectrum uses
    # seed + 1 = 7071): the exact top right singular vector, so step 0 breaks
    # down (beta = 0) and REQUIRE(kOk) cannot hold. Seed 7072 is the
    # non-degenerate version of the same test.
    lz = O.Lanczos(O.DenseOracle(X), 40, O.gaussian_matrix(n, 1, 7072)[:, 0], 3)
    events, worst_ident, worst_orth, fails = 0, 0.0, 0.0, 0
    slack = 2 * EPS * np.sqrt(n)
    for _ in range(40):
        info = lz.step(O.Options(omega=1e-8, omega_recurrence=recurrence), spec[0])
        assert info.status == 0
        events += info.reorthogonalized_left + info.reorthogonalized_right
        U, V = lz.left_basis(), lz.right_basis()
        j = U.shape[1]
        worst_ident = max(worst_ident, ident_defect(X, lz))
        worst_orth = max(worst_orth, np.abs(U.T @ U - np.eye(j)).max(),
                         np.abs(V.T @ V - np.eye(j + 1)).max())
        nu = np.ctypeslib.as_array(lz.f.nu, shape=(j,))
        mu = np.ctypeslib.as_array(lz.f.mu, shape=(j + 1,))
        fails += int(np.sum(nu[: j - 1] + slack < np.abs(U[:, : j - 1].T @ U[:, j - 1])))
        fails += int(np.sum(mu[:j] + slack < np.abs(V[:, :j].T @ V[:, j])))
    return events, worst_ident, worst_orth, fails


def test_partial_reorth_contract_complete_recurrence():  # :124-171
    events, ident, orth, fails = _run_partial(1)
    assert events >= 1 and ident <= 1e-10 and orth <= 1e-6 and fails == 0


def test_partial_reorth_contract_literal_recurrence():
    events, ident, orth, fails = _run_partial(0)
    assert events >= 1 and ident <= 1e-10 and orth <= 1e-6 and fails == 0


def test_degenerate_reference_start_breaks_down():
    X, spec, n = _decaying_case()
    lz = O.Lanczos(O.DenseOracle(X), 40, O.gaussian_matrix(n, 1, 7071)[:, 0], 3)
    assert lz.step(O.Options(omega=1e-8), spec[0]).status == 2


def test_literal_recurrence_documented_gap():
    """gkl.cpp:127-136 as written omits the |coupling|*nu term of the left
    omega recurrence. On the reference's own PRO solve (test_gkl.cpp:279-306)
    the estimates then under-run the true loss of orthogonality and the solve
    fails; the complete recurrence (default) passes.
    Pinned so the literal mode stays literal."""
    X = O.gaussian_matrix(120, 90, 909)
    s = np.linalg.svd(X, compute_uv=False)
    lit = O.svdl(O.DenseOracle(X), O.Options(k=10, tol=1e-10, seed=6, omega_recurrence=0))
    com = O.svdl(O.DenseOracle(X), O.Options(k=10, tol=1e-10, seed=6, omega_recurrence=1))
    assert not lit.all_converged and np.max(np.abs(lit.singvals - s[:10])) > 1e-6 * s[0]
    assert com.all_converged and np.max(np.abs(com.singvals - s[:10])) <= 1e-10 * s[0]


def test_rank_one():  # :173-193
    u = O.gaussian_matrix(30, 1, 51)[:, 0]
    v = O.gaussian_matrix(40, 1, 52)[:, 0]
    X = 7.0 * np.outer(u / np.linalg.norm(u), v / np.linalg.norm(v))
    r = O.svdl(O.DenseOracle(X), O.Options(k=1, tol=1e-8, seed=99))
    assert abs(r.singvals[0] - 7) <= 7e-12 and r.mvps <= 4 and r.all_converged
    assert np.linalg.norm(X @ r.V[:, 0] - r.singvals[0] * r.U[:, 0]) <= 7e-12


def test_diag_exact():  # :195-212
    r = O.svdl(O.DenseOracle(np.diag([5.0, 4, 3, 2, 1])), O.Options(k=5, tol=1e-10, seed=3, reorth=0))
    assert np.allclose(r.singvals, [5, 4, 3, 2, 1], rtol=1e-12) and r.mvps <= 12
    assert np.all(r.err <= 1e-12) and np.all(r.converged)


def test_thick_restart_preserves_ritz():  # :214-250
    X = O.gaussian_matrix(30, 40, 606)
    scale = np.linalg.svd(X, compute_uv=False)[0]
    lz = O.Lanczos(O.DenseOracle(X), 15, O.gaussian_matrix(40, 1, 607)[:, 0], 4)
    for _ in range(10):
        assert lz.step(full(), scale).status == 0
    before = lz.ritz(0.0)[0]
    lz.thick_restart(9)
    assert lz.steps == 9 and ident_defect(X, lz) <= 1e-10 * scale
    assert np.allclose(lz.ritz(0.0)[0][:9], before[:9], rtol=1e-12)
    for _ in range(4):
        assert lz.step(full(), scale).status == 0
        assert ident_defect(X, lz) <= 1e-10 * scale
    with pytest.raises(ValueError):
        lz.thick_restart(lz.steps + 1)


def test_restarted_plain_dense():  # :252-277
    X = O.gaussian_matrix(80, 100, 808)
    s = np.linalg.svd(X, compute_uv=False)
    d = O.DenseOracle(X)
    a = O.svdl(d, O.Options(k=5, tol=1e-10, reorth=0, seed=5))
    b = O.svdl(d, O.Options(k=5, tol=1e-10, reorth=0, seed=5, restart=1, max_subspace=20, keep=10))
    assert np.max(np.abs(a.singvals - s[:5])) <= 1e-8 * s[0]
    assert np.max(np.abs(b.singvals - s[:5])) <= 1e-8 * s[0] and b.restarts >= 1


def test_partial_solve_dense():  # :279-306
    X = O.gaussian_matrix(120, 90, 909)
    s = np.linalg.svd(X, compute_uv=False)
    r = O.svdl(O.DenseOracle(X), O.Options(k=10, tol=1e-10, seed=6))
    assert r.all_converged and np.max(np.abs(r.singvals - s[:10])) <= 1e-10 * s[0]
    for i in range(10):
        assert np.linalg.norm(X @ r.V[:, i] - r.singvals[i] * r.U[:, i]) <= 1e-10 * s[0] + 1e-12 * s[0]
    # test_gkl.cpp:298-299 also bounds the adjoint residual by tol*sigma_1; the
    # algorithm does not guarantee it (convergence uses the gap-refined
    # estimate, the adjoint residual is the crude coupling). Pinned as found:
    adj = max(np.linalg.norm(X.T @ r.U[:, i] - r.singvals[i] * r.V[:, i]) for i in range(10))
    assert adj > 1e-10 * s[0]


def test_error_bounds():  # :308-321
    X = O.gaussian_matrix(40, 60, 111)
    s = np.linalg.svd(X, compute_uv=False)
    r = O.svdl(O.DenseOracle(X), O.Options(k=8, tol=1e-9, seed=7))
    assert r.all_converged and np.all(np.abs(r.singvals - s[:8]) <= r.err + 1e-10)


def test_replay_budget_validation_zero():  # :336-403
    X = O.gaussian_matrix(60, 45, 222)
    o = O.Options(k=6, tol=1e-9, seed=314, record_history=True)
    a, b = O.svdl(O.DenseOracle(X), o), O.svdl(O.DenseOracle(X), o)
    assert all(np.array_equal(x, y) for x, y in zip(a.ritz_history, b.ritz_history))
    r = O.svdl(O.DenseOracle(O.gaussian_matrix(100, 80, 333)), O.Options(k=10, tol=1e-12, max_mvps=8, seed=1))
    assert not r.all_converged and r.mvps <= 8 and r.singvals.size == min(10, r.steps)
    for kw in [dict(k=9), dict(k=0), dict(k=2, tol=0.0),
               dict(k=2, restart=1, max_subspace=6, keep=6), dict(k=2, restart=1, max_subspace=6, keep=1),
               dict(k=2, restart=1, max_subspace=100, keep=4)]:
        with pytest.raises(ValueError):
            O.validate(O.Options(**kw), 10, 8)
    r = O.svdl(O.DenseOracle(np.zeros((6, 5))), O.Options(k=1, seed=11))
    assert r.mvps <= 16


def test_acceptance_criteria_1_2():  # acceptance.cpp:97-156
    worst = {0: 0.0, 1: 0.0}
    for t in range(20):
        m, n = 60 + (t * 37) % 241, 60 + (t * 53) % 341
        X = O.gaussian_matrix(m, n, 1000 + t)
        sigma = np.linalg.svd(X, compute_uv=False)[:10]
        d = O.DenseOracle(X)
        fro = O.Options(k=10, tol=1e-9, reorth=0, restart=1, max_subspace=40, keep=20, seed=t + 1)
        pro = O.Options(k=10, tol=1e-11, reorth=1, omega=1e-8, seed=t + 1)
        for idx, (opts, bar) in enumerate(((fro, 1e-8), (pro, 1e-10))):
            r = O.svdl(d, opts)
            assert r.singvals.size == 10
            dev = np.abs(r.singvals - sigma)
            worst[idx] = max(worst[idx], float(np.max(dev / sigma)))
            assert np.all(dev / sigma <= bar), (t, idx)
            assert np.all(dev[r.converged] <= r.err[r.converged] + 1e-10)
            assert r.err.sum() >= dev.sum() - 1e-9


# ------------------------------------------------------------ genio (test_genio.cpp)
def test_decode_kat():  # :64-78
    assert list(O.bed_decode(np.array([0x1B], np.uint8), 1, 4)[0]) == [0, 1, 3, 2]


def test_pads_ignored():  # :80-91
    assert O.bed_decode(np.array([0xFC], np.uint8), 1, 1)[0, 0] == 2


def test_roundtrip_and_stride():  # :93-124
    r = np.random.default_rng(99)
    d = r.integers(0, 4, size=(7, 13)).astype(np.uint8)
    b = O.bed_encode(d)
    stride = (13 + 3) // 4
    assert b.size == 7 * stride
    for i in range(7):
        assert (b[(i + 1) * stride - 1] >> 2) == 0
    assert np.array_equal(O.bed_decode(b, 7, 13), d)
    assert O.bed_encode(np.zeros((3, 5), np.uint8)).size == 3 * 2


def test_impute_standardize_semantics():  # :190-269
    # impute_mean: row [0, 2, missing] -> mean 1 ; all-missing -> 0
    d = np.array([[0, 2, 3], [3, 3, 3], [1, 1, 2]], np.uint8)
    c = O.marker_counts(O.bed_encode(d), 3, 3)
    assert c.tolist() == [[1, 0, 1, 1], [0, 0, 0, 3], [0, 2, 1, 0]]
    mu, inv_s = O.marker_scaling(c, 3, 0)
    assert mu[0] == 1.0 and mu[1] == 0.0 and inv_s[1] == 0.0
    # unit variance on [0, 2]: mean 1, population sd 1 -> entries -1, +1
    mu, inv_s = O.marker_scaling(O.marker_counts(O.bed_encode(np.array([[0, 2]], np.uint8)), 1, 2), 2, 0)
    assert mu[0] == 1.0 and inv_s[0] == 1.0
    # binomial on [0, 2]: p = 0.5 -> scale 0.5
    mu, inv_s = O.marker_scaling(O.marker_counts(O.bed_encode(np.array([[0, 2]], np.uint8)), 1, 2), 2, 1)
    assert abs(1.0 / inv_s[0] - 0.5) <= 1e-16
    # constant marker zeroed and flagged
    mu, inv_s = O.marker_scaling(O.marker_counts(O.bed_encode(np.full((1, 3), 2, np.uint8)), 1, 3), 3, 0)
    assert inv_s[0] == 0.0
    # every scaled row is centered over the mean-imputed row
    r = np.random.default_rng(314)
    d = r.integers(0, 4, size=(20, 31)).astype(np.uint8)
    pay = O.bed_encode(d)
    for scheme in (0, 1, 2):
        mu, inv_s = O.marker_scaling(O.marker_counts(pay, 20, 31), 31, scheme)
        g = O.GenoOracle(pay, 20, 31, mu, inv_s)
        assert np.abs(g.apply(np.ones(31))).max() <= 1e-12 * 31


def test_packed_operator_matches_dense_standardized():
    """The packed oracle equals the reference pipeline impute_mean ->
    standardize -> DenseOperator on the dense matrix (genio.cpp:124-185)."""
    r = np.random.default_rng(5)
    p, n = 40, 57
    d = r.integers(0, 3, size=(p, n)).astype(np.uint8)
    d[r.random((p, n)) < 0.1] = 3
    d[3, :] = 1
    pay = O.bed_encode(d)
    for scheme in (0, 1):
        mu, inv_s = O.marker_scaling(O.marker_counts(pay, p, n), n, scheme)
        # literal reference pipeline in numpy
        obs = d != 3
        dd = d.astype(float)
        means = np.array([dd[i, obs[i]].mean() if obs[i].any() else 0.0 for i in range(p)])
        imp = np.where(obs, dd, means[:, None])
        rm = imp.mean(axis=1)
        var = ((imp - rm[:, None]) ** 2).sum(axis=1) / n
        if scheme == 0:
            sc = np.sqrt(var)
        else:
            cl = 1.0 / (2.0 * n + 2.0)
            q = np.clip(rm / 2.0, cl, 1 - cl)
            sc = np.sqrt(q * (1 - q))
        Xs = np.where(var[:, None] == 0.0, 0.0, (imp - rm[:, None]) / np.where(sc == 0, 1, sc)[:, None])
        g = O.GenoOracle(pay, p, n, mu, inv_s)
        x = r.standard_normal(n)
        assert np.abs(g.apply(x) - Xs @ x).max() <= 1e-12 * np.abs(Xs).max() * np.sqrt(n)
        y = r.standard_normal(p)
        assert np.abs(g.apply_adjoint(y) - Xs.T @ y).max() <= 1e-12 * np.abs(Xs).max() * np.sqrt(p)


def test_packed_operator_matches_dense_none():
    """Scheme none = the reference CLI's --standardize none: the operator is
    impute_mean's matrix itself (missing -> observed row mean, all-missing
    row -> 0; genio.cpp:124-148, gkpca.cpp:89-103), not centered."""
    r = np.random.default_rng(6)
    p, n = 40, 57
    d = r.integers(0, 3, size=(p, n)).astype(np.uint8)
    d[r.random((p, n)) < 0.15] = 3
    d[2, :] = 3
    pay = O.bed_encode(d)
    mu, inv_s = O.marker_scaling(O.marker_counts(pay, p, n), n, 3)
    assert np.all(mu == 0.0) and np.all(inv_s == 1.0)
    obs = d != 3
    dd = d.astype(float)
    means = np.array([dd[i, obs[i]].mean() if obs[i].any() else 0.0 for i in range(p)])
    imp = np.where(obs, dd, means[:, None])
    g = O.GenoOracle(pay, p, n, mu, inv_s)
    x = r.standard_normal(n)
    assert np.abs(g.apply(x) - imp @ x).max() <= 1e-12 * np.sqrt(n) * 2
    y = r.standard_normal(p)
    assert np.abs(g.apply_adjoint(y) - imp.T @ y).max() <= 1e-12 * np.sqrt(p) * 2


def test_oracle_threads_deterministic():
    r = np.random.default_rng(1)
    p, n = 300, 1001
    d = r.integers(0, 4, size=(p, n)).astype(np.uint8)
    pay = O.bed_encode(d)
    mu, inv_s = O.marker_scaling(O.marker_counts(pay, p, n), n, 2)
    g1 = O.GenoOracle(pay, p, n, mu, inv_s, 1)
    g4 = O.GenoOracle(pay, p, n, mu, inv_s, 4)
    x, y = r.standard_normal(n), r.standard_normal(p)
    assert np.array_equal(g1.apply(x), g4.apply(x))
    assert np.array_equal(g1.apply_adjoint(y), g4.apply_adjoint(y))
