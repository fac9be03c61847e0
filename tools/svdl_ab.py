"""A/B timing of whole svdl solves: median of R solves (after one warm-up)
on a BASELINE config, printed as one JSON line. GKB_LIB selects the build.

usage: svdl_ab.py [config] [reps]
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg), scheme=gkb.ScalingScheme.kHwe)
opts = synth.config_options(cfg)
gkb.svdl(op, opts)
walls, devs = [], []
for _ in range(reps):
    t0 = time.perf_counter()
    res = gkb.svdl(op, opts)
    walls.append(time.perf_counter() - t0)
    devs.append(res.stats.device_seconds)
s = res.stats
print(json.dumps(dict(lib=os.path.basename(os.environ.get("GKB_LIB", "libgkb.so")), config=cfg,
                      wall_med=round(statistics.median(walls), 5), wall_min=round(min(walls), 5),
                      dev_med=round(statistics.median(devs), 5), mvps=s.mvps, restarts=s.restarts,
                      sigma1=float(res.singvals[0]))))
