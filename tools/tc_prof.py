"""Short driver for an ncu capture of the tcgen05 block kernel: config 4,
apply_block with k = 16 (GKB_TC_BLOCK=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GKB_TC_BLOCK"] = "1"
import numpy as np
import paper_1808_03374_b200 as gkb
from paper_1808_03374_b200 import synth
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg), scheme=gkb.ScalingScheme.kHwe)
X = np.random.default_rng(0).standard_normal((op.cols(), k))
for _ in range(2):
    op.apply_block(X)
print("ok")
