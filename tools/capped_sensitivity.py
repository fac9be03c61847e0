"""How well-posed is a CAPPED (unconverged) svdl result? GPU only, no oracle.

tools/full_parity.py CONFIG OUT MAX_MVPS compares the GPU's and the oracle's
truncated solves. At a cap the trailing Ritz triplets are not converged, and
the right Ritz vectors still carry part of the start vector's component in
null(X) (the right space has cols = n > rank when n > p, as in config 4), so
the k-dimensional right Ritz subspace of a truncated run moves with rounding
far more than its singular values or its left subspace do. This script shows
that with two GPU solves of the same operator that differ ONLY in rounding:
missing-data corrections summed as fp64 lists (GKB_MISS_MODE=list) or as exact
integer indicator sums (GKB_MISS_MODE=ind). For the capped and the converged
solve it reports per-sigma differences, subspace angles (all k, and the lead
both runs flag converged), each vector's misalignment, and -- the point --
|X d| / (sigma_k |d|) for the part d of the second run's right vectors outside
the first run's right Ritz subspace: ~0 means the difference lies in null(X)
and cannot change X v = sigma u.

usage: capped_sensitivity.py CONFIG OUT.json MAX_MVPS
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

import paper_1808_03374_b200 as gkb  # noqa: E402
from conftest import principal_angles  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/c{cfg}_capped_sensitivity.json"
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 420
spec = synth.config_spec(cfg)
base = synth.config_options(cfg)
k = int(base.k)


def solves(mode):
    os.environ["GKB_MISS_MODE"] = mode
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    capped = gkb.svdl(op, dataclasses.replace(base, max_mvps=cap))
    full = gkb.svdl(op, base)
    return op, capped, full


def unit_cols(M):
    return M / np.linalg.norm(M, axis=0)


def compare(a, b, op):
    ca, cb = np.asarray(a.converged, bool), np.asarray(b.converged, bool)
    lead = 0
    while lead < k and ca[lead] and cb[lead]:
        lead += 1
    Ua, Ub, Va, Vb = unit_cols(a.U), unit_cols(b.U), unit_cols(a.V), unit_cols(b.V)
    r = dict(
        mvps=[int(a.stats.mvps), int(b.stats.mvps)],
        restarts=[int(a.stats.restarts), int(b.stats.restarts)],
        converged_lead=lead,
        sigma_rel_diff_each=[float(abs(x - y) / abs(y)) for x, y in zip(a.singvals, b.singvals)],
        err_estimates=[float(x) for x in a.err_estimates],
        angle_U=float(principal_angles(Ua, Ub)),
        angle_V=float(principal_angles(Va, Vb)),
        angle_U_lead=float(principal_angles(Ua[:, :lead], Ub[:, :lead])) if lead else None,
        angle_V_lead=float(principal_angles(Va[:, :lead], Vb[:, :lead])) if lead else None,
        misalign_U_each=[float(1.0 - min(1.0, abs(Ua[:, i] @ Ub[:, i]))) for i in range(k)],
        misalign_V_each=[float(1.0 - min(1.0, abs(Va[:, i] @ Vb[:, i]))) for i in range(k)],
    )
    # the part of run b's right vectors outside run a's right Ritz subspace
    Qa = np.linalg.qr(Va)[0]
    D = Vb - Qa @ (Qa.T @ Vb)
    dn = np.linalg.norm(D, axis=0)
    XD = op.apply_block(np.asfortranarray(D))
    r["V_outside_norm_each"] = [float(x) for x in dn]
    r["X_outside_over_sigma_each"] = [float(np.linalg.norm(XD[:, i]) / (a.singvals[i] * dn[i])) if dn[i] > 0 else 0.0
                                      for i in range(k)]
    # same for the left side (X^T d / sigma |d|), for contrast
    Qu = np.linalg.qr(Ua)[0]
    E = Ub - Qu @ (Qu.T @ Ub)
    r["U_outside_norm_each"] = [float(x) for x in np.linalg.norm(E, axis=0)]
    return r


op_l, cap_l, full_l = solves("list")
op_l.close()
op_i, cap_i, full_i = solves("ind")
res = dict(
    config=synth.CONFIG_TEXT[cfg] if hasattr(synth, "CONFIG_TEXT") else cfg,
    options=synth.OPTIONS_TEXT[cfg] if hasattr(synth, "OPTIONS_TEXT") else "",
    k=k, max_mvps=cap, rows=int(spec.p), cols=int(spec.n),
    runs="GKB_MISS_MODE=list vs GKB_MISS_MODE=ind (same operator, products differ by rounding only)",
    capped=compare(cap_l, cap_i, op_i),
    converged=compare(full_l, full_i, op_i),
)
op_i.close()
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
