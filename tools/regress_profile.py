import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1808_03374_b200 as gkb
from paper_1808_03374_b200 import synth, regress as R
op = gkb.GenotypeOperator.from_synth(synth.config_spec(2), scheme=gkb.ScalingScheme.kHwe)
n = op.cols(); rng = np.random.default_rng(0)
y = rng.standard_normal(n); Z = rng.standard_normal((n, 10))
C = np.hstack([y[:, None], np.ones((n, 1)), Z])
op.apply_block(C)
def t(f, k=5):
    f(); s = time.perf_counter()
    for _ in range(k): f()
    return (time.perf_counter() - s) / k * 1e3
print("apply_block 12 cols %.2f ms" % t(lambda: op.apply_block(C)))
print("counts %.2f ms" % t(op.counts))
print("scaling %.2f ms" % t(op.scaling))
print("marker_sumsq %.2f ms" % t(lambda: R.marker_sumsq(op)))
print("constant_markers %.2f ms" % t(lambda: R.constant_markers(op)))
print("marker_scan %.2f ms" % t(lambda: R.marker_scan(op, y, Z)))
