"""Summarize an `ncu --set full` report into the JSON kept under profiles/.

usage: ncu_summary.py REPORT.ncu-rep OUT.json

Keys are short kernel names ("k_pm_main<0>" = K1 apply, "k_pm_main<1>" = K2
adjoint, ...); values are the metrics below as "value unit" strings. The
per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) is what
bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_barrier",
]


def short_name(full: str) -> str:
    m = re.search(r"::(\w+)(<[^>]*>)?\(", full)
    if not m:
        return full[:40]
    name = m.group(1)
    targs = m.group(2) or ""
    targs = re.sub(r"\(int\)", "", targs)
    return name + targs


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    res = {}
    for r in data:
        name = short_name(r[col["Kernel Name"]])
        if name in res:
            continue
        res[name] = {m: f"{r[col[m]]} {units[col[m]]}".strip() for m in METRICS if m in col}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v.get("gpu__time_duration.sum") for k, v in res.items()}))


if __name__ == "__main__":
    main()
