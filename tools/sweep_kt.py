"""Sweep the column-range width kt_cta (GKB_KT_CTA) of the packed products:
per-product main-kernel time for K1 (apply) and K2 (adjoint).

usage: sweep_kt.py config iters kt [kt ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, ROOT)
    import paper_1808_03374_b200 as gkb
    from paper_1808_03374_b200 import synth
    cfg, iters = int(sys.argv[2]), int(sys.argv[3])
    op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg), scheme=gkb.ScalingScheme.kHwe)
    op.bench(2, 5, flush_l2=False)
    k1 = op.bench(0, iters, flush_l2=False)
    k2 = op.bench(1, iters, flush_l2=False)
    print(f"  K1 step {k1[0]*1e3:7.2f} us main {k1[1]*1e3:7.2f} us | "
          f"K2 step {k2[0]*1e3:7.2f} us main {k2[1]*1e3:7.2f} us")
    sys.exit(0)
cfg, iters = sys.argv[1], sys.argv[2]
for kt in sys.argv[3:]:
    print(f"config {cfg} kt_cta {kt}", flush=True)
    subprocess.run([sys.executable, __file__, "--one", cfg, iters],
                   env=dict(os.environ, GKB_KT_CTA=kt), check=True)
