"""Prints the kernel sequence of two steady-state steps of an svdl solve from a
trace_svdl.py chrome trace: start / end relative to a K1 main launch.

usage: trace_step.py trace.json [k1_index]
"""
import json
import re
import sys

ev = [e for e in json.load(open(sys.argv[1]))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
k1 = [i for i, e in enumerate(ev) if "k_pm_main<0" in e["name"]]
j = int(sys.argv[2]) if len(sys.argv) > 2 else len(k1) // 2
i0, i1 = k1[j], k1[min(j + 2, len(k1) - 1)]
t0 = ev[i0]["ts"]
prev_end = None
for e in ev[i0:i1 + 1]:
    m = re.search(r"(k_\w+(<[^>]*>)?)", e["name"])
    n = m.group(1) if m else e["name"][:30]
    end = e["ts"] - t0 + e["dur"]
    inc = "" if prev_end is None else f"{end - prev_end:7.2f}"
    print(f"{e['ts'] - t0:9.2f} {end:9.2f} {e['dur']:7.2f} {inc:>7} {n}")
    prev_end = end if prev_end is None else max(prev_end, end)
