import os, sys, dataclasses
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1808_03374_b200 as gkb
from paper_1808_03374_b200 import synth
spec = synth.config_spec(2, scale=0.05)
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme(2))
base = synth.config_options(2)
R, T = gkb.ReorthMode, gkb.RestartMode
vs = [base, dataclasses.replace(base, reorth=R.kFull), dataclasses.replace(base, one_sided=True),
      dataclasses.replace(base, omega_recurrence=0), dataclasses.replace(base, omega=1e-4),
      dataclasses.replace(base, restart=T.kNone, max_mvps=120)]
for i, o in enumerate(vs):
    for host in ("1", "0"):
        os.environ["GKB_HOST_STEP"] = host
        r = gkb.svdl(op, o)
        print(i, "host" if host == "1" else "dev ", r.singvals[:3], r.stats.mvps, r.stats.steps, r.stats.restarts, r.stats.reorth_count, r.stats.host_syncs, flush=True)
