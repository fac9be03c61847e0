"""Timing of the widened rows on config 2: subspace iteration (per iteration:
block products vs host QR/condition) and the per-marker regression scan."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import regress as R  # noqa: E402
from paper_1808_03374_b200 import subspace as S  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

spec = synth.config_spec(2)
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
k = 10
Y = np.random.default_rng(0).standard_normal((spec.p, k))
Yf = np.asfortranarray(Y)
op.apply_adjoint_block(Yf)
t = time.perf_counter()
for _ in range(5):
    Z = op.apply_adjoint_block(Yf)
    W = op.apply_block(Z)
tb = (time.perf_counter() - t) / 5
t = time.perf_counter()
for _ in range(5):
    Q = S.qr_thin(W)[0]
    c = S.basis_condition(Q)
tq = (time.perf_counter() - t) / 5
print(f"subspace pass (k={k}): block products {tb*1e3:.2f} ms, host qr+condition {tq*1e3:.2f} ms")
t = time.perf_counter()
r = S.subspace_iterate(op, k, S.SubspaceVariant.kQr, 1e-8, 40, 0)
ts = time.perf_counter() - t
print(f"subspace_iterate k={k} 40 iters max: {ts:.3f} s, iterations {r.state.iterations}, "
      f"mvps {r.mvps}, converged {r.converged}, last delta {r.state.delta_history[-1]:.2e}")
y = np.random.default_rng(1).standard_normal(spec.n)
Zpc = gkb.svdl(op, gkb.GklOptions(k=k, tol=1e-8)).V
t = time.perf_counter()
scan = R.marker_scan(op, y, Zpc)
tr = time.perf_counter() - t
print(f"marker_scan p={spec.p} k={k}: {tr*1e3:.1f} ms ({spec.p / tr / 1e6:.2f} M markers/s)")
