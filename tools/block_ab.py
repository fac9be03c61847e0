"""A/B helper: two-column block products (k_pm_main2) on one config, device
time per apply_block / apply_adjoint_block of 4 columns (host arrays; the
kernels dominate at config 4). GKB_LIB selects the build.

usage: block_ab.py CONFIG [reps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = synth.config_spec(cfg)
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
rng = np.random.default_rng(0)
X = rng.standard_normal((spec.n, 4))
U = rng.standard_normal((spec.p, 4))
op.apply_block(X)
op.apply_adjoint_block(U)
t0 = time.perf_counter()
for _ in range(reps):
    op.apply_block(X)
t1 = time.perf_counter()
for _ in range(reps):
    op.apply_adjoint_block(U)
t2 = time.perf_counter()
lib = os.path.basename(os.environ.get("GKB_LIB", "libgkb.so"))
print(f"{lib:18s} cfg {cfg}: apply_block(4) {(t1-t0)/reps*1e3:8.2f} ms  "
      f"apply_adjoint_block(4) {(t2-t1)/reps*1e3:8.2f} ms", flush=True)
