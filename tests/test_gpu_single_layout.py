"""Single-layout mode: a shard whose two tile layouts do
not fit in HBM (config 5 at 2 GPUs: 125 GB per layout per GPU) keeps layout 1
only and reads the adjoint (reference apply_adjoint, X^T y, linop.hpp:55-58)
from it (k_pm_adj_l1). GKB_LAYOUTS=1 forces the mode at operator build; the
products and solves must match the oracle exactly as the two-layout path
does."""
import os

import numpy as np
import pytest

from conftest import principal_angles, rel_err, sigma_rel_err

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1), (5, 17), (33, 100), (130, 257), (257, 1000), (1031, 2049), (64, 4099),
          (1792, 3), (1793, 1791), (3600, 1100), (100, 9000)]


def _payload(p, n, seed, missing):
    from paper_1808_03374_b200 import genio
    rng = np.random.default_rng(seed)
    d = rng.integers(0, 3, size=(p, n)).astype(np.uint8)
    d[rng.random((p, n)) < missing] = 3
    if p >= 3:
        d[0, :] = 3
        d[1, :] = 2
    return genio.encode(d)


@pytest.mark.parametrize("p,n", SHAPES)
@pytest.mark.parametrize("missing", [0.0, 0.01, 0.05])
def test_adjoint_single_layout_vs_oracle(gkb, orc, monkeypatch, p, n, missing):
    monkeypatch.setenv("GKB_LAYOUTS", "1")
    payload = _payload(p, n, 17 + p + n, missing)
    op = gkb.GenotypeOperator.from_bed_payload(payload, p, n, scheme=gkb.ScalingScheme.kHwe)
    assert op.modes()[0] == 1
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, p, n, mu, inv_s)
    rng = np.random.default_rng(5)
    for scale in (1.0, 1e-200, 1e150):
        y = rng.standard_normal(p) * scale
        za, zo = op.apply_adjoint(y), ref.apply_adjoint(y)
        assert np.max(np.abs(za - zo)) <= 1e-12 * max(1e-300, np.max(np.abs(zo))) + \
            1e-13 * scale * np.sqrt(p) * (np.max(inv_s) * 2.0 + 1.0)
        x = rng.standard_normal(n) * scale
        assert rel_err(op.apply(x), ref.apply(x)) <= 1e-12 or np.max(np.abs(ref.apply(x))) == 0


@pytest.mark.parametrize("cfg,scale", [(2, 0.05), (3, 0.01), (4, 0.01), (5, 0.005)])
def test_svdl_single_layout_vs_oracle(gkb, orc, monkeypatch, cfg, scale):
    from paper_1808_03374_b200 import synth
    monkeypatch.setenv("GKB_LAYOUTS", "1")
    spec = synth.config_spec(cfg, scale=scale)
    opts = synth.config_options(cfg)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    assert op.modes()[0] == 1
    payload = orc.synth_bed(spec)
    mu, inv_s = op.scaling()
    g = gkb.svdl(op, opts)
    o = orc.svdl(orc.GenoOracle(payload, spec.p, spec.n, mu, inv_s, nthreads=8),
                 orc.Options.from_gkl(opts))
    assert sigma_rel_err(g.singvals, o.singvals) <= 1e-9
    assert principal_angles(g.U, o.U) < 1e-6 and principal_angles(g.V, o.V) < 1e-6
    assert abs(g.stats.restarts - o.restarts) <= 1


def test_single_equals_dual_config2(gkb, monkeypatch):
    from paper_1808_03374_b200 import synth
    spec = synth.config_spec(2)
    y = np.random.default_rng(3).standard_normal(spec.p)
    monkeypatch.setenv("GKB_LAYOUTS", "2")
    op2 = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    z2 = op2.apply_adjoint(y)
    b2 = op2.info()["device_bytes"]
    op2.close()
    monkeypatch.setenv("GKB_LAYOUTS", "1")
    op1 = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    assert op1.modes()[0] == 1
    assert rel_err(op1.apply_adjoint(y), z2) <= 1e-14
    assert op1.info()["device_bytes"] < 0.7 * b2


@pytest.mark.slow
def test_config5_subblock_single_layout_vs_golden(gkb, monkeypatch):
    import hashlib
    from paper_1808_03374_b200 import synth
    monkeypatch.setenv("GKB_LAYOUTS", "1")
    ref = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                               "c5_sub_100k.npz"))
    spec = synth.config_spec(5).sub_block(100_000, 100_000)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    assert op.modes()[0] == 1
    g = gkb.svdl(op, synth.config_options(5))
    assert sigma_rel_err(g.singvals, ref["singvals"]) <= 1e-9
    assert principal_angles(g.U, ref["U"].astype(np.float64)) < 1e-6
    assert principal_angles(g.V, ref["V"].astype(np.float64)) < 1e-6
    assert abs(g.stats.restarts - int(ref["restarts"])) <= 1
