"""Packed genotype operator on the B200 vs the CPU oracle (through the C ABI).

Covers: layout round trip (.bed bytes back from HBM), device marker counts
and (mu, 1/s) bit-exact against the oracle, K1 (apply, X x) and K2
(apply_adjoint, X^T y) against the oracle's packed operator on ragged
shapes, missing entries, all-missing and zero-variance markers, adjoint
consistency (linop.cpp:30-39), sharded == unsharded, and the device
generator's bytes == the CPU generator's bytes.
"""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def random_payload(p, n, seed, missing=0.02, special_rows=True):
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 3, size=(p, n)).astype(np.uint8)
    d[rng.random((p, n)) < missing] = 3
    if special_rows and p >= 4:
        d[0, :] = 3                 # all missing
        d[1, :] = 2                 # zero variance
        d[2, :] = np.where(rng.random(n) < 0.5, 1, 3)  # one observed dosage + missing
    from paper_1808_03374_b200 import genio
    return genio.encode(d), d


SHAPES = [(1, 1), (4, 16), (5, 17), (7, 3), (33, 100), (130, 257), (257, 1000), (1031, 2049),
          (64, 4099),
          # column-range boundaries (14 tiles = 1792 columns; the unrolled full-range loop)
          (5, 1792), (5, 1793), (1792, 3), (1793, 1791),
          # >= 65,536 samples: the adjoint's thread-per-sample finish (k2_reduce_seq)
          (37, 70001)]


@pytest.mark.parametrize("p,n", SHAPES)
def test_layout_roundtrip_and_counts(gkb, orc, p, n):
    payload, d = random_payload(p, n, seed=p * 1000 + n)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=None)
    back = op.read_bed()
    assert np.array_equal(back, payload)
    assert np.array_equal(op.counts(), orc.marker_counts(payload, p, n))


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_scaling_bit_exact(gkb, orc, scheme):
    p, n = 300, 517
    payload, _ = random_payload(p, n, seed=11)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme(scheme))
    mu, inv_s = op.scaling()
    mu_o, is_o = orc.marker_scaling(orc.marker_counts(payload, p, n), n, scheme)
    assert np.array_equal(mu, mu_o)
    assert np.array_equal(inv_s, is_o)


@pytest.mark.parametrize("p,n", SHAPES)
@pytest.mark.parametrize("missing", [0.0, 0.05])
def test_apply_and_adjoint_vs_oracle(gkb, orc, p, n, missing):
    payload, _ = random_payload(p, n, seed=7 + p + n, missing=missing)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, p, n, mu, inv_s)
    rng = np.random.default_rng(3)
    for scale in (1.0, 1e-200, 1e150):
        x = rng.standard_normal(n) * scale
        y = rng.standard_normal(p) * scale
        ya, yo = op.apply(x), ref.apply(x)
        za, zo = op.apply_adjoint(y), ref.apply_adjoint(y)
        # fp64 summation-order differences only (tolerance relative to the
        # magnitude of the summed terms, ~ sqrt(n) * eps * |x|_inf * max|entry|)
        assert np.max(np.abs(ya - yo)) <= 1e-12 * max(1e-300, np.max(np.abs(yo))) + \
            1e-13 * scale * np.sqrt(n) * (np.max(inv_s) * 2.0 + 1.0)
        assert np.max(np.abs(za - zo)) <= 1e-12 * max(1e-300, np.max(np.abs(zo))) + \
            1e-13 * scale * np.sqrt(p) * (np.max(inv_s) * 2.0 + 1.0)


@pytest.mark.parametrize("missing", [0.01, 0.013])
def test_tall_sample_count_lists_vs_oracle(gkb, orc, missing):
    """n >= 65,536 with per-CTA missing lists (list mode): K2's partials are
    summed by the thread-per-sample finish, K1's and K2's list walks take the
    uniform chunk loop; both against the oracle."""
    p, n = 41, 70003
    payload, _ = random_payload(p, n, seed=91, missing=missing)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, p, n, mu, inv_s)
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal(n), rng.standard_normal(p)
    ya, yo = op.apply(x), ref.apply(x)
    za, zo = op.apply_adjoint(y), ref.apply_adjoint(y)
    assert np.max(np.abs(ya - yo)) <= 1e-12 * np.max(np.abs(yo))
    assert np.max(np.abs(za - zo)) <= 1e-12 * np.max(np.abs(zo))


def test_edge_rows_are_zero(gkb, orc):
    p, n = 9, 50
    payload, d = random_payload(p, n, seed=5)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kUnitVariance)
    mu, inv_s = op.scaling()
    assert inv_s[0] == 0.0 and mu[0] == 0.0     # all missing: mean 0, flagged
    assert inv_s[1] == 0.0 and mu[1] == 2.0     # constant marker zeroed (genio.cpp:167-171)
    assert inv_s[2] == 0.0 and mu[2] == 1.0
    y = op.apply(np.ones(n))
    assert y[0] == 0.0 and y[1] == 0.0 and y[2] == 0.0


def test_adjoint_consistency(gkb):
    p, n = 211, 389
    payload, _ = random_payload(p, n, seed=9)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n)
    rng = np.random.default_rng(1)
    u, v = rng.standard_normal(p), rng.standard_normal(n)
    mis = abs(u @ op.apply(v) - op.apply_adjoint(u) @ v) / (np.linalg.norm(u) * np.linalg.norm(v))
    assert mis <= 1e-12


@pytest.mark.parametrize("nshards", [2, 3, 5])
def test_sharded_equals_unsharded(gkb, orc, nshards):
    p, n = 1003, 777
    payload, _ = random_payload(p, n, seed=21)
    one = gkb.GenotypeOperator.from_bed_payload(payload, p, n)
    ctx = gkb.Context([0] * nshards)
    sh = gkb.GenotypeOperator.from_bed_payload(payload, p, n, ctx=ctx)
    assert np.array_equal(sh.read_bed(), payload)
    assert np.array_equal(sh.counts(), one.counts())
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal(n), rng.standard_normal(p)
    # apply is shard-local: identical bytes per row
    assert np.array_equal(sh.apply(x), one.apply(x))
    # adjoint sums shard partials: fp64 reassociation only
    assert rel_err(sh.apply_adjoint(y), one.apply_adjoint(y)) <= 1e-13


def test_mvp_counter(gkb):
    payload, _ = random_payload(8, 40, seed=1)
    op = gkb.GenotypeOperator.from_bed_payload(payload, 8, 40)
    op.apply(np.ones(40))
    op.apply_adjoint(np.ones(8))
    op.apply(np.ones(40))
    assert op.mvps() == 3
    with pytest.raises(ValueError):
        op.apply(np.ones(8))


def test_synth_bytes_match_cpu_generator(gkb, orc):
    from paper_1808_03374_b200 import synth
    for cfg in (1, 2, 3, 4):
        spec = synth.config_spec(cfg, scale=0.02)
        op = gkb.GenotypeOperator.from_synth(spec, scheme=None)
        cpu = orc.synth_bed(spec)
        assert np.array_equal(op.read_bed(), cpu), cfg


def test_format_errors(gkb):
    with pytest.raises(gkb.FormatError):
        gkb.GenotypeOperator.from_bed_payload(np.zeros(10, np.uint8), 3, 16)
    with pytest.raises(ValueError):
        gkb.GenotypeOperator.from_bed_payload(np.zeros(0, np.uint8), 0, 16)


@pytest.mark.parametrize("p,n", [(257, 1000), (3001, 5003)])
def test_pinned_buffers_and_out(gkb, p, n):
    """gkb.pinned_empty + out= (page-locked host vectors, used in place by the
    kernels: K1's finish fused into the last CTA of each row block) give the
    same bits as pageable numpy vectors (staged copies, separate reduce) --
    also with several column ranges and row blocks; out= validation follows
    the reference's invalid_argument behaviour (ValueError)."""
    payload, _ = random_payload(p, n, seed=5)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    x = np.random.default_rng(1).standard_normal(n)
    xp = gkb.pinned_empty(n)
    xp[:] = x
    yp = gkb.pinned_empty(p)
    zp = gkb.pinned_empty(n)
    y = op.apply(x)
    assert op.apply(xp, out=yp) is yp
    assert np.array_equal(y, yp)
    z = op.apply_adjoint(y)
    op.apply_adjoint(yp, out=zp)
    assert np.array_equal(z, zp)
    with pytest.raises(ValueError):
        op.apply(x, out=np.empty(p + 1))
    with pytest.raises(ValueError):
        op.apply(x, out=np.empty(p, dtype=np.float32))


@pytest.mark.parametrize("scheme", [0, 1, 3])
def test_schemes_vs_oracle(gkb, orc, scheme):
    """unit / binomial / none (the reference CLI's mean-imputed raw matrix:
    missing -> observed row mean) against the oracle, with missing entries and
    all-missing / zero-variance rows."""
    p, n = 1031, 2049
    payload, _ = random_payload(p, n, seed=17 + scheme, missing=0.05)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme(scheme))
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, p, n, mu, inv_s)
    x = np.random.default_rng(scheme).standard_normal(n)
    assert rel_err(op.apply(x), ref.apply(x)) <= 1e-12
    y = np.random.default_rng(scheme + 10).standard_normal(p)
    assert rel_err(op.apply_adjoint(y), ref.apply_adjoint(y)) <= 1e-12


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_block_products_equal_single_columns(gkb, k):
    """Block products (two columns per pass through the shared-expansion
    kernel, an odd last column alone; the default below 6 columns)
    give each column bit for bit the single-vector product, with
    missing entries, several column ranges and row blocks."""
    p, n = 3001, 5003
    payload, _ = random_payload(p, n, seed=23, missing=0.03)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    rng = np.random.default_rng(k)
    X = rng.standard_normal((n, k))
    Y = op.apply_block(X)
    for c in range(k):
        assert np.array_equal(Y[:, c], op.apply(X[:, c])), c
    U = rng.standard_normal((p, k))
    Z = op.apply_adjoint_block(U)
    for c in range(k):
        assert np.array_equal(Z[:, c], op.apply_adjoint(U[:, c])), c


@pytest.mark.parametrize("nshards,p", [(2, 3001), (3, 7)])
def test_block_products_sharded(gkb, nshards, p):
    """Two-column block products on a multi-shard context (rows split across
    shards, possibly tiny or empty shards; the adjoint summed across shards)
    equal the single-shard operator's columns bit for bit."""
    n = 2051
    payload, _ = random_payload(p, n, seed=31, missing=0.03)
    one = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    ctx = gkb.Context([0] * nshards)
    sh = gkb.GenotypeOperator.from_bed_payload(payload, p, n, ctx=ctx,
                                               scheme=gkb.ScalingScheme.kHwe)
    rng = np.random.default_rng(nshards)
    X = rng.standard_normal((n, 4))
    U = rng.standard_normal((p, 4))
    assert np.array_equal(sh.apply_block(X), one.apply_block(X))
    Za, Zb = sh.apply_adjoint_block(U), one.apply_adjoint_block(U)
    # the adjoint's cross-shard sum adds per-shard partials (order differs from one shard)
    assert np.max(np.abs(Za - Zb)) <= 1e-12 * np.max(np.abs(Zb))


def test_norm_estimate_and_adjoint_mismatch_vs_oracle(gkb, orc):
    """norm_estimate / adjoint_mismatch (linop.cpp:9-39) on the device operator
    against the oracle's restatement on the same payload and scaling."""
    p, n = 1201, 903
    payload, _ = random_payload(p, n, seed=41, missing=0.02)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, p, n, mu, inv_s, nthreads=4)
    a, b = gkb.norm_estimate(op, 20), orc.norm_estimate(ref, 20)
    assert abs(a - b) <= 1e-11 * b
    assert gkb.adjoint_mismatch(op) <= 1e-14 and orc.adjoint_mismatch(ref) <= 1e-14


@pytest.mark.parametrize("k", [3, 4, 5, 8, 11, 12, 16, 17])
@pytest.mark.parametrize("p,n,missing", [(3001, 5003, 0.03), (257, 1000, 0.0), (64, 4099, 0.2)])
def test_tc_block_products_vs_oracle(gkb, orc, monkeypatch, k, p, n, missing):
    """Block products of k >= 3 columns on the 5th-generation tensor cores
    (k_pm_blk_tc: tcgen05.mma kind::i8, accumulators in TMEM, exact
    indicator-MMA missing corrections; at most 16 columns per pass) against
    the oracle, column by column, and against the single-vector products."""
    monkeypatch.setenv("GKB_TC_BLOCK", "1")
    payload, _ = random_payload(p, n, seed=41 + k + p, missing=missing)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, p, n, mu, inv_s)
    rng = np.random.default_rng(k + n)
    X = rng.standard_normal((n, k)) * np.logspace(-3, 3, k)
    Y = op.apply_block(X)
    U = rng.standard_normal((p, k)) * np.logspace(2, -2, k)
    Z = op.apply_adjoint_block(U)
    for c in range(k):
        yo, zo = ref.apply(X[:, c]), ref.apply_adjoint(U[:, c])
        assert np.max(np.abs(Y[:, c] - yo)) <= 1e-12 * max(1e-300, np.max(np.abs(yo))), c
        assert np.max(np.abs(Z[:, c] - zo)) <= 1e-12 * max(1e-300, np.max(np.abs(zo))), c
        assert rel_err(Y[:, c], op.apply(X[:, c])) <= 1e-13
        assert rel_err(Z[:, c], op.apply_adjoint(U[:, c])) <= 1e-13


def test_tc_block_products_in_subspace_iteration(gkb, orc, monkeypatch):
    """The tcgen05 block products inside an iterative solver (back-to-back
    PDL-chained launches, both directions): subspace iteration on the
    config-2 model equals the two-columns-per-pass path."""
    from paper_1808_03374_b200 import subspace as Sb
    from paper_1808_03374_b200 import synth
    spec = synth.config_spec(2, scale=0.05)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    monkeypatch.setenv("GKB_TC_BLOCK", "0")
    a = Sb.subspace_iterate(op, 6, Sb.SubspaceVariant.kQr, 1e-9, 100, 1)
    monkeypatch.setenv("GKB_TC_BLOCK", "1")
    b = Sb.subspace_iterate(op, 6, Sb.SubspaceVariant.kQr, 1e-9, 100, 1)
    from conftest import principal_angles, sigma_rel_err
    assert sigma_rel_err(b.singvals, a.singvals) <= 1e-9
    assert principal_angles(b.basis, a.basis) < 1e-6
    assert abs(a.state.iterations - b.state.iterations) <= 1
