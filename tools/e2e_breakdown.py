"""Where the host-buffer (e2e) step time goes on config 2: the two public
calls vs their device-resident work vs bare pinned copies of the same sizes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

spec = synth.config_spec(2)
op = gkb.GenotypeOperator.from_synth(spec, scheme=gkb.ScalingScheme.kHwe)
x = gkb.pinned_empty(spec.n)
x[:] = np.random.default_rng(7).standard_normal(spec.n)
y = gkb.pinned_empty(spec.p)
z = gkb.pinned_empty(spec.n)


def timeit(f, k=200):
    for _ in range(10):
        f()
    t = time.perf_counter()
    for _ in range(k):
        f()
    return (time.perf_counter() - t) / k * 1e6


print(f"apply (host bufs)         {timeit(lambda: op.apply(x, out=y)):8.1f} us")
print(f"apply_adjoint (host bufs) {timeit(lambda: op.apply_adjoint(y, out=z)):8.1f} us")
st, mn, _ = op.bench(0, 200, flush_l2=False)
print(f"apply device-resident     {st*1e3:8.1f} us (main {mn*1e3:.1f})")
st, mn, _ = op.bench(1, 200, flush_l2=False)
print(f"adjoint device-resident   {st*1e3:8.1f} us (main {mn*1e3:.1f})")
dx = torch.empty(spec.n, dtype=torch.float64, device="cuda")
dy = torch.empty(spec.p, dtype=torch.float64, device="cuda")
hx = torch.from_numpy(x)
hy = torch.from_numpy(y)


def copies():
    dx.copy_(hx, non_blocking=True)
    hy.copy_(dy, non_blocking=True)
    torch.cuda.synchronize()


def copies_big():
    dy.copy_(hy, non_blocking=True)
    hy.copy_(dy, non_blocking=True)
    torch.cuda.synchronize()


print(f"H2D 80KB + D2H 800KB      {timeit(copies):8.1f} us")
print(f"H2D 800KB + D2H 800KB     {timeit(copies_big):8.1f} us")
print(f"sync only                 {timeit(torch.cuda.synchronize):8.1f} us")
