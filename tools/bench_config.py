"""Supplementary measurement of another BASELINE config on one GPU (bench.py's
contract line stays config 2): device-resident K1+K2 step GB/s, the main
kernels' roofline fraction against MEASURED_PEAKS.json, and time to the top-k
triplets with that config's BASELINE options. One JSON line.

usage: bench_config.py CONFIG [steps]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
spec = synth.config_spec(cfg)
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
b = spec.p * ((spec.n + 3) // 4)
op.bench(2, 3, flush_l2=False)
step_ms, _, _ = op.bench(2, steps, flush_l2=False)
k1 = op.bench(0, steps, flush_l2=False)[1]
k2 = op.bench(1, steps, flush_l2=False)[1]
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
opts = synth.config_options(cfg)
gkb.svdl(op, opts)  # warm-up (pools, staging)
t0 = time.perf_counter()
res = gkb.svdl(op, opts)
tts = time.perf_counter() - t0
dom = max(k1, k2)
print(json.dumps({
    "config": cfg, "n": spec.n, "p": spec.p, "packed_bytes": b, "steps": steps,
    "value_gbs": round(2 * b / (step_ms * 1e-3) / 1e9, 1), "ms_per_step": round(step_ms, 4),
    "k1_main_ms": round(k1, 4), "k2_main_ms": round(k2, 4),
    "roofline": {"achieved": round(b / (dom * 1e-3) / 1e9, 1), "peak": peak,
                 "frac": round(b / (dom * 1e-3) / 1e9 / peak, 4)},
    "time_to_solution": {"seconds": round(tts, 4), "mvps": res.stats.mvps,
                         "restarts": res.stats.restarts, "converged": res.stats.converged,
                         "k": opts.k, "host_syncs": res.stats.host_syncs},
}))
