"""Main-kernel time of the packed products against the missing rate (VERDICT
r1 item 7). usage: missing_perf.py CONFIG [rates...]  -> one JSON line per rate"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rates = [float(r) for r in sys.argv[2:]] or [0.0, 0.01, 0.02, 0.05, 0.10]
for r in rates:
    spec = dataclasses.replace(synth.config_spec(cfg), missing_rate=r)
    op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
    b = spec.p * ((spec.n + 3) // 4)
    op.bench(2, 3, flush_l2=False)
    k1 = op.bench(0, 20, flush_l2=False)
    k2 = op.bench(1, 20, flush_l2=False)
    info = op.info()
    print(json.dumps({"config": cfg, "missing_rate": r, "nmissing": info["nmissing"],
                      "device_bytes": info["device_bytes"],
                      "k1_step_ms": round(k1[0], 5), "k1_main_ms": round(k1[1], 5),
                      "k2_step_ms": round(k2[0], 5), "k2_main_ms": round(k2[1], 5),
                      "k1_main_gbs": round(b / k1[1] / 1e6, 1),
                      "k2_main_gbs": round(b / k2[1] / 1e6, 1)}), flush=True)
    op.close()
