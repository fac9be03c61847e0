"""Two-column block products (k_pm_main2) vs two single products, device-resident."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

for cfg in (2, 3):
    op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg), scheme=gkb.ScalingScheme.kHwe)
    op.bench(3, 3, flush_l2=False)
    pair = op.bench(3, 30, flush_l2=False)[0]
    single = op.bench(2, 30, flush_l2=False)[0]
    b = op.packed_bytes() if hasattr(op, "packed_bytes") else None
    print(f"config {cfg}: 2 x (K1+K2) as singles {2 * single * 1e3:.1f} us, as column pairs "
          f"{pair * 1e3:.1f} us ({2 * single / pair:.2f}x)")
