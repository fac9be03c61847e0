"""BASELINE full sizes on the device (config 2: 10,000 x 100,000; config 4:
500,000 x 100,000 = 12.5 GB packed): full oracle parity where the CPU oracle
finishes in seconds (config 2), size-independent properties otherwise --
adjoint consistency, linearity, sharded == unsharded, bit-exact .bed
read-back and oracle agreement on sampled marker rows."""
import os

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _op(gkb, cfg, nshards=1):
    from paper_1808_03374_b200 import synth
    spec = synth.config_spec(cfg)
    ctx = gkb.Context([0] * nshards) if nshards > 1 else None
    return spec, gkb.GenotypeOperator.from_synth(spec, ctx=ctx, scheme=gkb.ScalingScheme.kHwe)


def test_config2_full_oracle_parity(gkb, orc):
    spec, op = _op(gkb, 2)
    payload = orc.synth_bed(spec)
    assert np.array_equal(op.counts(), orc.marker_counts(payload, spec.p, spec.n))
    rows = np.r_[0:64, spec.p - 64:spec.p]
    stride = (spec.n + 3) // 4
    back = op.read_bed().reshape(spec.p, stride)
    assert np.array_equal(back[rows], payload.reshape(spec.p, stride)[rows])
    mu, inv_s = op.scaling()
    ref = orc.GenoOracle(payload, spec.p, spec.n, mu, inv_s, nthreads=os.cpu_count() or 1)
    x = np.random.default_rng(0).standard_normal(spec.n)
    y = op.apply(x)
    assert rel_err(y, ref.apply(x)) <= 1e-12
    assert rel_err(op.apply_adjoint(y), ref.apply_adjoint(y)) <= 1e-12


def test_config4_full_properties(gkb, orc):
    spec, op = _op(gkb, 4)
    rng = np.random.default_rng(1)
    x, x2 = rng.standard_normal(spec.n), rng.standard_normal(spec.n)
    y = op.apply(x)
    z = op.apply_adjoint(y)
    # adjoint consistency <y, A x> = <A^T y, x> (linop.cpp:30-39)
    assert abs(y @ y - z @ x) <= 1e-12 * abs(y @ y)
    # linearity
    assert rel_err(op.apply(2.0 * x - 3.0 * x2), 2.0 * y - 3.0 * op.apply(x2)) <= 1e-12
    # sampled rows against the oracle (payload of just those markers)
    mu, inv_s = op.scaling()
    for j0 in (0, spec.p // 2, spec.p - 48):
        j1 = j0 + 48
        sub = orc.synth_bed(spec, j0, j1)
        ref = orc.GenoOracle(sub, j1 - j0, spec.n, mu[j0:j1], inv_s[j0:j1],
                             nthreads=os.cpu_count() or 1)
        assert rel_err(y[j0:j1], ref.apply(x)) <= 1e-12
        assert np.array_equal(op.read_bed(j0, j1 - j0).reshape(-1), sub.reshape(-1))


def test_config4_sharded_equals_unsharded(gkb):
    spec, op1 = _op(gkb, 4)
    x = np.random.default_rng(2).standard_normal(spec.n)
    y1 = op1.apply(x)
    z1 = op1.apply_adjoint(y1)
    op1.close()
    _, op2 = _op(gkb, 4, nshards=2)
    assert np.array_equal(op2.apply(x), y1)   # K1 is shard-local: bitwise
    assert rel_err(op2.apply_adjoint(y1), z1) <= 1e-14
