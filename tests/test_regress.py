"""Regression (regress.cpp / gkpca regress): the reference's test_regress.cpp
cases for ols_fit / pc_adjusted_fit, and the device per-marker scan against
the reference's per-marker QR loop (gkpca.cpp:620-668) on the dense matrix."""
import numpy as np
import pytest


@pytest.fixture
def R():
    from paper_1808_03374_b200 import regress
    return regress


def normal_eq(X, y):
    beta = np.linalg.solve(X.T @ X, X.T @ y)
    r = y - X @ beta
    s2 = r @ r / X.shape[0]
    return beta, s2, s2 * np.linalg.inv(X.T @ X)


def test_noise_free(R, orc):  # :17-26
    X = orc.gaussian_matrix(30, 4, 1201)
    beta = np.array([1.0, -2.0, 3.0, 0.5])
    f = R.ols_fit(X, X @ beta)
    assert np.abs(f.beta_hat - beta).max() <= 1e-12
    assert f.sigma2_hat <= 1e-24 and np.abs(f.residuals).max() <= 1e-12


def test_intercept_only(R):  # :28-35
    y = np.array([1.0, 2.0, 3.0, 4.0, 10.0])
    f = R.ols_fit(np.ones((5, 1)), y)
    assert abs(f.beta_hat[0] - 4.0) <= 1e-14
    assert abs(f.sigma2_hat - ((y - 4) ** 2).sum() / 5) <= 1e-13


def test_normal_equations_oracle(R, orc):  # :37-49
    for seed in (11, 12, 13):
        X = orc.gaussian_matrix(50, 3, seed)
        y = orc.gaussian_matrix(50, 1, seed + 100)[:, 0] + 2 * X[:, 0]
        f = R.ols_fit(X, y)
        b, s2, cov = normal_eq(X, y)
        assert np.abs(f.beta_hat - b).max() <= 1e-10
        assert abs(f.sigma2_hat - s2) <= 1e-10 * s2
        assert np.abs(f.cov_beta - cov).max() <= 1e-10 * np.abs(cov).max()


def test_variance_conventions(R, orc):  # :51-63
    X = orc.gaussian_matrix(40, 5, 77)
    y = orc.gaussian_matrix(40, 1, 78)[:, 0]
    b, u = R.ols_fit(X, y, False), R.ols_fit(X, y, True)
    assert abs(u.sigma2_hat - b.sigma2_hat * 40 / 35) <= 1e-15 * u.sigma2_hat
    rss = b.residuals @ b.residuals
    assert abs(b.sigma2_hat * 40 - rss) <= 4e-16 * rss
    assert np.abs(X.T @ b.residuals).max() <= 1e-10 * np.linalg.norm(y)


def test_rank_deficiency(R, orc):  # :65-94
    G = orc.gaussian_matrix(20, 3, 5150)
    y = orc.gaussian_matrix(20, 1, 5151)[:, 0]
    X = np.column_stack([G[:, 0], G[:, 1], G[:, 0], G[:, 2]])
    with pytest.raises(R.RankDeficiencyError) as e:
        R.ols_fit(X, y)
    assert e.value.column == 2
    Xc = np.column_stack([G[:, 0], G[:, 1], 0.5 * G[:, 0] - 2 * G[:, 1]])
    with pytest.raises(R.RankDeficiencyError) as e:
        R.ols_fit(Xc, y)
    assert e.value.column == 2


def test_shapes(R):  # :96-103
    for X, y in ((np.ones((5, 2)), np.ones(4)), (np.ones((5, 0)), np.ones(5)),
                 (np.ones((2, 3)), np.ones(2))):
        with pytest.raises(ValueError):
            R.ols_fit(X, y)


def test_pc_adjusted_block_oracle(R, orc):  # :105-120
    X, Z = orc.gaussian_matrix(60, 2, 900), orc.gaussian_matrix(60, 3, 901)
    y = orc.gaussian_matrix(60, 1, 902)[:, 0] + X[:, 1] - 0.5 * Z[:, 0]
    f = R.pc_adjusted_fit(X, Z, y)
    b, s2, cov = normal_eq(np.hstack([X, Z]), y)
    assert np.abs(f.beta_hat - b[:2]).max() <= 1e-10
    assert np.abs(f.gamma_hat - b[2:]).max() <= 1e-10
    assert abs(f.joint.sigma2_hat - s2) <= 1e-10 * s2
    assert np.abs(f.cov_beta - cov[:2, :2]).max() <= 1e-10 * np.abs(cov[:2, :2]).max()
    with pytest.raises(ValueError):
        R.pc_adjusted_fit(X, np.ones((59, 3)), y)


def test_orthogonal_adjustment(R, orc):  # :122-132
    from paper_1808_03374_b200.subspace import qr_thin
    Q = qr_thin(orc.gaussian_matrix(45, 5, 33))[0]
    X, Z = 3.0 * Q[:, :2], Q[:, 2:]
    y = orc.gaussian_matrix(45, 1, 34)[:, 0]
    assert np.abs(R.pc_adjusted_fit(X, Z, y).beta_hat - R.ols_fit(X, y).beta_hat).max() <= 1e-12


def test_null_marker_coverage(R, orc):  # :134-150
    covered = 0
    for t in range(1000):
        seed = 5000 + 7 * t
        Z, X = orc.gaussian_matrix(40, 2, seed), orc.gaussian_matrix(40, 1, seed + 1)
        y = Z @ np.array([1.0, -0.5]) + 0.3 * orc.gaussian_matrix(40, 1, seed + 2)[:, 0]
        f = R.pc_adjusted_fit(X, Z, y, True)
        covered += abs(f.beta_hat[0]) <= 3 * np.sqrt(f.cov_beta[0, 0])
    assert covered >= 950


# ---------------------------------------------------------------- device scan
def _reference_scan(R, M, Z, y, unbiased):
    """The reference loop (gkpca.cpp:620-668): X_i = [1, m_i], fit with Z."""
    n = M.shape[1]
    out = []
    for i in range(M.shape[0]):
        X = np.column_stack([np.ones(n), M[i]])
        try:
            f = R.pc_adjusted_fit(X, Z, y, unbiased) if Z.shape[1] else R.ols_fit(X, y, unbiased)
            cov = f.cov_beta
            s2 = f.joint.sigma2_hat if Z.shape[1] else f.sigma2_hat
            out.append((f.beta_hat[1], np.sqrt(cov[1, 1]), f.beta_hat[0], s2))
        except R.RankDeficiencyError as e:
            out.append(("err", e.column))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,k,unbiased", [(2, 3, False), (0, 0, True), (3, 2, False)])
def test_device_scan_vs_reference_loop(gkb, R, scheme, k, unbiased):
    from paper_1808_03374_b200 import genio
    rng = np.random.default_rng(scheme + k)
    p, n = 150, 120
    d = rng.binomial(2, rng.uniform(0.1, 0.9, size=(p, 1)), size=(p, n)).astype(np.uint8)
    d[rng.random((p, n)) < 0.02] = 3
    d[5, :] = 1                           # constant marker
    d[9, :] = np.where(rng.random(n) < 0.3, 3, 2)   # one observed value + missing
    op = gkb.GenotypeOperator.from_bed_payload(genio.encode(d), p, n,
                                               scheme=gkb.ScalingScheme(scheme))
    M = op.apply_block(np.eye(n))          # the operator's dense matrix (p x n)
    Z = np.linalg.qr(rng.standard_normal((n, k)))[0] if k else np.zeros((n, 0))
    y = rng.standard_normal(n) + (M[3] / max(1e-9, np.abs(M[3]).max()))
    scan = R.marker_scan(op, y, Z if k else None, unbiased)
    ref = _reference_scan(R, M, Z, y, unbiased)
    for i, r in enumerate(ref):
        if r[0] == "err":
            assert scan.dependent[i] and r[1] == 1, i
            continue
        assert not scan.dependent[i], i
        b, se, ic, s2 = r
        assert abs(scan.beta[i] - b) <= 1e-9 * max(1.0, abs(b)), i
        assert abs(scan.se[i] - se) <= 1e-9 * se, i
        assert abs(scan.intercept[i] - ic) <= 1e-9 * max(1.0, abs(ic)), i
        assert abs(scan.sigma2[i] - s2) <= 1e-9 * s2, i
    assert scan.dependent[5] and scan.dependent[9]


@pytest.mark.gpu
@pytest.mark.parametrize("k,unbiased", [(0, False), (3, True), (10, False)])
def test_device_marker_scan_matches_host_algebra(gkb, k, unbiased):
    """gkb_geno_marker_scan (block product + one thread per marker on the
    device) against the host Frisch-Waugh-Lovell algebra on the same block
    product (regress.marker_scan with explicit sumsq/constant)."""
    from paper_1808_03374_b200 import regress as R
    from paper_1808_03374_b200 import synth
    spec = synth.config_spec(2, scale=0.05)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    rng = np.random.default_rng(3 + k)
    y = rng.standard_normal(spec.n)
    Z = rng.standard_normal((spec.n, k)) if k else None
    dev = R.marker_scan(op, y, Z, unbiased)
    host = R.marker_scan(op, y, Z, unbiased, sumsq=R.marker_sumsq(op),
                         constant=R.constant_markers(op))
    assert np.array_equal(dev.dependent, host.dependent)
    ok = ~host.dependent
    for f in ("beta", "se", "intercept", "sigma2"):
        a, b = getattr(dev, f)[ok], getattr(host, f)[ok]
        assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) <= 1e-8, f


@pytest.mark.gpu
def test_device_marker_scan_sharded(gkb):
    """The device scan on a two-shard context gives every marker's fit exactly
    as on one shard (each marker's row lives on one shard)."""
    from paper_1808_03374_b200 import regress as R
    from paper_1808_03374_b200 import synth
    spec = synth.config_spec(2, scale=0.05)
    one = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    two = gkb.GenotypeOperator.from_synth(spec, ctx=gkb.Context([0, 0]),
                                          scheme=gkb.ScalingScheme.kHwe)
    rng = np.random.default_rng(9)
    y = rng.standard_normal(spec.n)
    Z = rng.standard_normal((spec.n, 4))
    a, b = R.marker_scan(one, y, Z), R.marker_scan(two, y, Z)
    assert np.array_equal(a.dependent, b.dependent)
    for f in ("beta", "se", "intercept", "sigma2"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
