"""Robustness to missing data: the packed products and
the full svdl at 1-50% missing entries against the oracle. Above ~1.8%
missing a CTA block's list no longer fits the shared-memory staging
(kEntCap) and the main kernels walk it in global memory; both paths must
give the oracle's results (impute_mean semantics, genio.cpp:124-148:
a missing entry contributes the observed row mean, i.e. 0 after centering).
"""
import dataclasses

import numpy as np
import pytest

from conftest import principal_angles, rel_err, sigma_rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("missing", [0.01, 0.02, 0.05, 0.10, 0.5])
def test_products_vs_oracle_missing_rates(gkb, orc, missing):
    from paper_1808_03374_b200 import synth
    spec = dataclasses.replace(synth.config_spec(2, scale=0.3), missing_rate=missing)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    payload = orc.synth_bed(spec)
    assert np.array_equal(op.counts(), orc.marker_counts(payload, spec.p, spec.n))
    frac = op.counts()[:, 3].sum() / (spec.p * spec.n)
    assert abs(frac - missing) < 0.01 * max(missing, 0.01) + 2e-3
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, spec.p, spec.n, mu, inv_s, nthreads=8)
    rng = np.random.default_rng(4)
    x = rng.standard_normal(spec.n)
    y = op.apply(x)
    assert rel_err(y, ref.apply(x)) <= 1e-12
    assert rel_err(op.apply_adjoint(y), ref.apply_adjoint(y)) <= 1e-12


@pytest.mark.parametrize("missing", [0.02, 0.05, 0.10])
def test_svdl_vs_oracle_missing_rates(gkb, orc, missing):
    from paper_1808_03374_b200 import synth
    spec = dataclasses.replace(synth.config_spec(2, scale=0.05), missing_rate=missing)
    opts = synth.config_options(2)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    payload = orc.synth_bed(spec)
    mu, inv_s = op.scaling()
    g = gkb.svdl(op, opts)
    o = orc.svdl(orc.GenoOracle(payload, spec.p, spec.n, mu, inv_s, nthreads=8),
                 orc.Options.from_gkl(opts))
    assert sigma_rel_err(g.singvals, o.singvals) <= 1e-9
    assert principal_angles(g.U, o.U) < 1e-6 and principal_angles(g.V, o.V) < 1e-6
    assert abs(g.stats.restarts - o.restarts) <= 1
