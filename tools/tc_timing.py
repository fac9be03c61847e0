"""Block products of k columns: tcgen05 one-pass kernel (k_pm_blk_tc) vs the
two-columns-per-pass mma.sync kernel (GKB_TC_BLOCK=0), on a BASELINE config,
through the widened rows that use them (subspace iteration, regression scan)
and the host-API block products. One JSON line per mode.
usage: tc_timing.py CONFIG"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import regress as Rg  # noqa: E402
from paper_1808_03374_b200 import subspace as Sb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = synth.config_spec(cfg)
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
b = spec.p * ((spec.n + 3) // 4)
rng = np.random.default_rng(1)
for mode in ("1", "0"):
    os.environ["GKB_TC_BLOCK"] = mode
    out = {"config": cfg, "tc": mode == "1"}
    for k in (4, 12, 16):
        X = rng.standard_normal((spec.n, k))
        U = rng.standard_normal((spec.p, k))
        op.apply_block(X)
        op.apply_adjoint_block(U)
        t0 = time.perf_counter()
        for _ in range(3):
            op.apply_block(X)
        ta = (time.perf_counter() - t0) / 3
        t0 = time.perf_counter()
        for _ in range(3):
            op.apply_adjoint_block(U)
        tz = (time.perf_counter() - t0) / 3
        out[f"k{k}"] = {"apply_block_s": round(ta, 5), "adjoint_block_s": round(tz, 5),
                        "apply_gbs_per_vector": round(k * b / ta / 1e9, 1),
                        "adjoint_gbs_per_vector": round(k * b / tz / 1e9, 1)}
    Sb.subspace_iterate(op, 10, Sb.SubspaceVariant.kQr, 1e-8, 4, 0)
    t0 = time.perf_counter()
    sres = Sb.subspace_iterate(op, 10, Sb.SubspaceVariant.kQr, 1e-8, 40, 0)
    out["subspace_k10_40it_s"] = round(time.perf_counter() - t0, 4)
    out["subspace_mvps"] = sres.mvps
    pheno = rng.standard_normal(spec.n)
    Z = rng.standard_normal((spec.n, 10))
    Rg.marker_scan(op, pheno, Z)
    t0 = time.perf_counter()
    Rg.marker_scan(op, pheno, Z)
    out["marker_scan_s"] = round(time.perf_counter() - t0, 5)
    print(json.dumps(out), flush=True)
