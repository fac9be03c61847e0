import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1808_03374_b200 as gkb
from paper_1808_03374_b200 import synth
os.environ["GKB_TC_BLOCK"] = "1"
which = sys.argv[1]; k = int(sys.argv[2])
cfg, scale = (2, 0.05)
op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg, scale=scale), scheme=gkb.ScalingScheme.kHwe)
rng = np.random.default_rng(0)
try:
    if which == "a":
        op.apply_block(rng.standard_normal((op.cols(), k)))
    else:
        op.apply_adjoint_block(rng.standard_normal((op.rows(), k)))
    print(which, k, "ok", flush=True)
except Exception as e:
    print(which, k, "FAIL", str(e)[:80], flush=True)
