"""One-off: the reference's literal CPU path on the FULL config 2 (10,000 x
100,000; the dense standardized fp64 matrix is 8 GB), 1 thread as the
reference runs (bench.py cpu_dense_svdl, which the default bench run times on
config 1 only), beside the GPU solve of the same config. Run on the GPU box;
the JSON goes under profiles/.

usage: cpu_dense_c2.py OUT.json
"""
import json
import os
import sys
import time

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)

import bench  # noqa: E402
import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cpu_dense_c2.json"
W = bench.load_workloads()
cpu = bench.cpu_dense_svdl(W, 2)
op = gkb.GenotypeOperator.from_synth(synth.config_spec(2), scheme=gkb.ScalingScheme.kHwe)
opts = synth.config_options(2)
gkb.svdl(op, opts)
t0 = time.perf_counter()
g = gkb.svdl(op, opts)
cpu.update(gpu_seconds=round(time.perf_counter() - t0, 4), gpu_mvps=g.stats.mvps,
           gpu_restarts=g.stats.restarts, gpu_sigma_1=float(g.singvals[0]),
           sigma_1_rel_diff=abs(float(g.singvals[0]) - cpu["sigma_1"]) / cpu["sigma_1"],
           host_cores_available=os.cpu_count())
with open(out, "w") as f:
    json.dump(cpu, f, indent=1)
print(json.dumps(cpu))
