"""One-off svdl parity at a FULL BASELINE config size (config 3: 6.25 GB,
~15 min of oracle on 16 cores; config 4: 12.5 GB, ~2 h) with the BASELINE
options: the GPU solve against the CPU oracle's solve on the same seeded .bed
bytes and scaling, with the protocol of tests/test_gpu_parity_full.py
(per-sigma 1e-9, principal angles < 1e-6, restarts +-1). Too slow for the
test suite; run on the GPU box, result committed under profiles/.

usage: full_parity.py CONFIG OUT.json [MAX_MVPS]

MAX_MVPS caps both solves at the same mvp budget (GklOptions::max_mvps): the
GPU and the oracle then run the same truncated trajectory, which is how config
4's full size fits the GPU box's one-hour call limit (the uncapped oracle solve
takes ~2 h on 16 cores). At a cap the trailing Ritz triplets are not converged
(config 4's sigma_4.. sit at the edge of the Marchenko-Pastur bulk, gaps of
2e-4 relative), so the k-dimensional Ritz subspace is not yet a well-posed
quantity: the record then also holds the angles over the leading triplets BOTH
solvers flag converged, each vector's own misalignment, and the error
estimates -- `pass` uses the converged lead for the angles and all k values for
sigma.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
import paper_1808_03374_b200 as gkb  # noqa: E402
from conftest import principal_angles, sigma_rel_err  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/c{cfg}_parity.json"
spec = synth.config_spec(cfg)
opts = synth.config_options(cfg)
max_mvps = int(sys.argv[3]) if len(sys.argv) > 3 else None
if max_mvps:
    opts.max_mvps = max_mvps
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
mu, inv_s = op.scaling()
t0 = time.perf_counter()
g = gkb.svdl(op, opts)
t_gpu = time.perf_counter() - t0
op.close()
t0 = time.perf_counter()
payload = orc.synth_bed(spec)
t_gen = time.perf_counter() - t0
nt = os.cpu_count() or 1
t0 = time.perf_counter()
o = orc.svdl(orc.GenoOracle(payload, spec.p, spec.n, mu, inv_s, nthreads=nt),
             orc.Options.from_gkl(opts))
t_cpu = time.perf_counter() - t0
res = dict(
    config=synth.CONFIG_TEXT[cfg] if hasattr(synth, "CONFIG_TEXT") else cfg,
    options=synth.OPTIONS_TEXT[cfg] if hasattr(synth, "OPTIONS_TEXT") else "",
    k=int(opts.k),
    max_mvps=max_mvps,
    sigma_rel_err_each=[float(abs(a - b) / abs(b)) for a, b in zip(g.singvals, o.singvals)],
    sigma_gpu=[float(x) for x in g.singvals],
    sigma_oracle=[float(x) for x in o.singvals],
    sigma_rel_err_max=float(sigma_rel_err(g.singvals, o.singvals)),
    angle_U=float(principal_angles(g.U, o.U)),
    angle_V=float(principal_angles(g.V, o.V)),
    mvps_gpu=int(g.stats.mvps), mvps_oracle=int(o.mvps),
    restarts_gpu=int(g.stats.restarts), restarts_oracle=int(o.restarts),
    converged_gpu=bool(g.stats.converged), converged_oracle=bool(o.all_converged),
    seconds_gpu=round(t_gpu, 3), seconds_oracle=round(t_cpu, 1), oracle_threads=nt,
    seconds_oracle_generate=round(t_gen, 1),
    thresholds=dict(sigma_rel=1e-9, angle=1e-6, restarts=1),
)
gc, oc = np.asarray(g.converged, bool), np.asarray(o.converged, bool)
lead = 0
while lead < int(opts.k) and gc[lead] and oc[lead]:
    lead += 1
res["converged_lead"] = lead
res["converged_flags_equal"] = bool(np.array_equal(gc, oc))
res["err_estimates_gpu"] = [float(x) for x in g.err_estimates]
res["err_estimates_oracle"] = [float(x) for x in o.err]
res["misalign_U_each"] = [float(1.0 - min(1.0, abs(np.dot(g.U[:, i], o.U[:, i]))
                                             / (np.linalg.norm(g.U[:, i]) * np.linalg.norm(o.U[:, i]))))
                           for i in range(int(opts.k))]
res["misalign_V_each"] = [float(1.0 - min(1.0, abs(np.dot(g.V[:, i], o.V[:, i]))
                                             / (np.linalg.norm(g.V[:, i]) * np.linalg.norm(o.V[:, i]))))
                           for i in range(int(opts.k))]
if max_mvps and lead < int(opts.k):
    res["angle_U_lead"] = float(principal_angles(g.U[:, :lead], o.U[:, :lead])) if lead else None
    res["angle_V_lead"] = float(principal_angles(g.V[:, :lead], o.V[:, :lead])) if lead else None
    aU, aV = res["angle_U_lead"] or 0.0, res["angle_V_lead"] or 0.0
else:
    aU, aV = res["angle_U"], res["angle_V"]
res["pass"] = (res["sigma_rel_err_max"] <= 1e-9 and aU < 1e-6 and aV < 1e-6
               and res["converged_flags_equal"]
               and abs(res["restarts_gpu"] - res["restarts_oracle"]) <= 1
               and res["converged_gpu"] == res["converged_oracle"])
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res))
