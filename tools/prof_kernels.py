"""Short driver for ncu captures of the packed kernels (K1 apply, K2 adjoint)
on the bench workload (BASELINE config 2, device-generated)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg), scheme=gkb.ScalingScheme.kHwe)
t = op.bench(2, iters, flush_l2=False)
print(f"config {cfg}: step {t[0]:.4f} ms, main kernels {t[1]:.4f} ms")
