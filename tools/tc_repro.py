import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1808_03374_b200 as gkb
from paper_1808_03374_b200 import synth
step = sys.argv[1]
op = gkb.GenotypeOperator.from_synth(synth.config_spec(3, scale=0.01), scheme=gkb.ScalingScheme.kHwe)
print("modes", op.modes(), "p n", op.rows(), op.cols(), flush=True)
rng = np.random.default_rng(0)
X = rng.standard_normal((op.cols(), 3))
if step in ("apply", "both"):
    Y = op.apply_block(X); gkb.default_context().synchronize(); print("apply_block ok", flush=True)
    y = op.apply(X[:, 0]); print("apply ok", np.max(np.abs(y - Y[:, 0])), flush=True)
if step in ("adj", "both"):
    U = rng.standard_normal((op.rows(), 3))
    Z = op.apply_adjoint_block(U); gkb.default_context().synchronize(); print("adjoint_block ok", flush=True)
    z = op.apply_adjoint(U[:, 0]); print("adjoint ok", np.max(np.abs(z - Z[:, 0])), flush=True)
