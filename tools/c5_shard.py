"""Config 5 at 2 GPUs, the per-GPU shard on one B200: the seeded leading
500,000 SNPs x 1,000,000 samples of config 5 (rank 0's rows under
gkb_partition_rows at G = 2; 125 GB packed). Two layouts do not fit in HBM,
so the layout plan keeps layout 1 (single-layout mode). Reports the plan,
the device bytes, the K1 / K2 main-kernel and step times, and a bounded
svdl sample with config 5's options. One JSON line.

usage: c5_shard.py [steps] [max_mvps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses  # noqa: E402

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
max_mvps = int(sys.argv[2]) if len(sys.argv) > 2 else 120
full = synth.config_spec(5)
spec = full.sub_block(500_000, 1_000_000)
t0 = time.perf_counter()
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
gkb.default_context().synchronize()
t_build = time.perf_counter() - t0
layouts, dense = op.modes()
info = op.info()
b = spec.p * ((spec.n + 3) // 4)
op.bench(2, 1, flush_l2=False)
k1 = op.bench(0, steps, flush_l2=False)
k2 = op.bench(1, steps, flush_l2=False)
st = op.bench(2, steps, flush_l2=False)
opts = dataclasses.replace(synth.config_options(5), max_mvps=max_mvps)
t0 = time.perf_counter()
res = gkb.svdl(op, opts)
t_svdl = time.perf_counter() - t0
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps({
    "workload": "config 5 at G=2, rank-0 shard: 500,000 SNPs x 1,000,000 samples (125 GB packed)",
    "plan": gkb.geno_plan(spec.p, spec.n, 0.01, 178 << 30),
    "layouts": layouts, "dense_missing": dense, "device_bytes": info["device_bytes"],
    "nmissing": info["nmissing"], "build_seconds": round(t_build, 2),
    "k1_main_ms": round(k1[1], 3), "k2_main_ms": round(k2[1], 3),
    "k1_main_gbs": round(b / k1[1] / 1e6, 1), "k2_main_gbs": round(b / k2[1] / 1e6, 1),
    "k1_frac": round(b / k1[1] / 1e6 / peak, 4), "k2_frac": round(b / k2[1] / 1e6 / peak, 4),
    "step_ms": round(st[0], 3), "step_gbs": round(2 * b / st[0] / 1e6, 1),
    "svdl_sample": {"max_mvps": max_mvps, "seconds": round(t_svdl, 3), "mvps": res.stats.mvps,
                    "steps": res.stats.steps, "sigma_1": float(res.singvals[0])
                    if res.singvals.size else None,
                    "solve_gbs": round(res.stats.mvps * b / t_svdl / 1e9, 1)},
}), flush=True)
