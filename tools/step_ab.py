"""A/B helper: step and main-kernel times of one config through gkb_op_bench
(device-resident, no flush), one line per run. GKB_LIB selects the build.

usage: step_ab.py CONFIG [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg), scheme=gkb.ScalingScheme.kHwe)
op.bench(2, 3, flush_l2=False)
k1s, k1m, _ = op.bench(0, iters, flush_l2=False)
k2s, k2m, _ = op.bench(1, iters, flush_l2=False)
st, _, _ = op.bench(2, iters, flush_l2=False)
lib = os.path.basename(os.environ.get("GKB_LIB", "libgkb.so"))
print(f"{lib:18s} cfg {cfg}: K1 step {k1s*1e3:8.1f} main {k1m*1e3:8.1f} | K2 step {k2s*1e3:8.1f} "
      f"main {k2m*1e3:8.1f} | K1+K2 {st*1e3:8.1f} us", flush=True)
