"""Kernel timeline of one svdl solve via the CUDA activity tracer that
torch.profiler wraps (no nsys in this image): per-kernel real durations and
the idle time between kernels (host round trips).

usage: trace_svdl.py [config] [out.json]
"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1808_03374_b200 as gkb  # noqa: E402
from paper_1808_03374_b200 import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = sys.argv[2] if len(sys.argv) > 2 else None
torch.cuda.init()
op = gkb.GenotypeOperator.from_synth(synth.config_spec(cfg), scheme=gkb.ScalingScheme.kHwe)
opts = synth.config_options(cfg)
gkb.svdl(op, opts)  # warm-up
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = gkb.svdl(op, opts)
print(f"device {res.stats.device_seconds*1e3:.2f} ms, host_syncs {res.stats.host_syncs}")
path = out or "/tmp/trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    name = e["name"].split("(")[0].replace("void ", "")[-40:]
    agg[(e["cat"], name)][0] += 1
    agg[(e["cat"], name)][1] += e["dur"]
busy = 0.0
end = ev[0]["ts"]
for e in ev:
    s, t = e["ts"], e["ts"] + e["dur"]
    if t > end:
        busy += t - max(s, end)
        end = t
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
print(f"span {span/1e3:.2f} ms, busy {busy/1e3:.2f} ms, idle {(span-busy)/1e3:.2f} ms, "
      f"{len(ev)} device ops")
for (cat, name), (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{d/1e3:8.2f} ms {n:6d}x {d/n:8.2f} us  {cat:10s} {name}")
