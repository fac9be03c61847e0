"""Runs svdl on a BASELINE config (device-generated) once and prints its
stats; used for ncu launch lists of the whole solve.

usage: svdl_run.py [config] [scale]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg, scale), scheme=gkb.ScalingScheme.kHwe)
opts = synth.config_options(cfg)
res = gkb.svdl(op, opts)  # warm-up
t0 = time.perf_counter()
res = gkb.svdl(op, opts)
wall = time.perf_counter() - t0
s = res.stats
print(f"config {cfg}: wall {wall:.4f} s (C {s.wall_seconds:.4f}), device {s.device_seconds:.4f} s, mvps {s.mvps}, steps "
      f"{s.steps}, restarts {s.restarts}, reorth {s.reorth_count}, host_syncs {s.host_syncs}")
