"""Summarise a chrome trace written by trace_svdl.py: per-kernel totals,
idle gaps, and one step of the timeline.

usage: trace_summary.py trace.json [nsample]
"""
import collections
import json
import re
import sys

ev = [e for e in json.load(open(sys.argv[1]))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
nsample = int(sys.argv[2]) if len(sys.argv) > 2 else 0


def nm(e):
    m = re.search(r"(k_\w+(<\d+>)?|k\d_\w+|Memcpy \w+|Memset)", e["name"])
    return m.group(1) if m else e["name"][:30]


agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    agg[nm(e)][0] += 1
    agg[nm(e)][1] += e["dur"]
for k, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{d/1e3:8.2f} ms {n:6d}x {d/n:8.2f} us {k}")
big, small, end = [], 0.0, None
for e in ev:
    if end is not None:
        g = e["ts"] - end
        if g >= 10:
            big.append(round(g))
        elif g > 0:
            small += g
    end = max(e["ts"] + e["dur"], end or 0)
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
print(f"span {span/1e3:.2f} ms; gaps >= 10 us: {sum(big)/1e3:.2f} ms ({len(big)}), "
      f"smaller gaps {small/1e3:.2f} ms")
i0 = len(ev) // 2
prev = None
for e in ev[i0:i0 + nsample]:
    gap = e["ts"] - prev if prev else 0
    print(f"gap {gap:7.1f}  dur {e['dur']:7.1f}  {nm(e)}")
    prev = e["ts"] + e["dur"]
