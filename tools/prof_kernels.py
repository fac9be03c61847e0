"""Short driver for timing / ncu captures of the packed products (K1 apply,
K2 adjoint) on a BASELINE config (device-generated).

usage: prof_kernels.py [config] [iters] [missing_rate]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = synth.config_spec(cfg)
if len(sys.argv) > 3:
    spec.missing_rate = float(sys.argv[3])
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
t = op.bench(2, iters, flush_l2=False)
print(f"config {cfg} (missing {spec.missing_rate}): step {t[0]:.4f} ms, main kernels {t[1]:.4f} ms")
