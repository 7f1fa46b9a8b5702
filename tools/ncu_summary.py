"""Summarise an ncu capture into the JSON files committed under profiles/.

    python tools/ncu_summary.py gpurun_out/TAG profiles/ROUND

reads TAG/launches.csv (the `--metrics gpu__time_duration.sum` launch list of the timed
steps) and TAG/prof.ncu-rep (the `--set full` capture), writes
ROUND_launches.json (every launch + per-kernel share of the step) and
ROUND_kernels.json (the metrics DESIGN.md cites, one row per captured launch).
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def launches(path):
    rows = []
    with open(path) as fh:
        text = fh.read()
    start = text.find('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Unit") == "usecond":
            ns *= 1e3
        elif r.get("Metric Unit") == "msecond":
            ns *= 1e6
        rows.append({"kernel": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"],
                     "ns": ns})
    own = [r for r in rows if "ef::" in r["kernel"]]
    tot = sum(r["ns"] for r in own) or 1.0
    per = defaultdict(lambda: [0, 0.0])
    for r in own:
        name = r["kernel"].split("(")[0].replace("void ", "")
        per[name][0] += 1
        per[name][1] += r["ns"]
    share = sorted(({"kernel": k, "launches": c, "ns": ns, "share": ns / tot} for k, (c, ns) in per.items()),
                   key=lambda x: -x["ns"])
    return {"launches": rows, "own_kernels_by_time": share, "own_total_ns": tot}


def kernels(rep):
    """rep: a .ncu-rep, or the `--page raw --csv` export of one (prof_raw.csv, written on the GPU
    box when the report itself is too large to bring back)."""
    if rep.endswith(".csv"):
        with open(rep) as fh:
            out = fh.read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                             capture_output=True, text=True, check=True).stdout
    rdr = list(csv.reader(io.StringIO(out)))
    head, units = rdr[0], rdr[1]
    rows = []
    for r in rdr[2:]:
        d = dict(zip(head, r))
        row = {"Kernel Name": d.get("Kernel Name")}
        for h, u in zip(head, units):
            if h in METRICS:
                row[f"{h} [{u}]" if u else h] = d[h]
        rows.append(row)
    return rows


def main():
    src, dst = sys.argv[1], sys.argv[2]
    with open(dst + "_launches.json", "w") as fh:
        json.dump(launches(src + "/launches.csv"), fh, indent=1)
    rep = src + "/prof.ncu-rep" if os.path.exists(src + "/prof.ncu-rep") else src + "/prof_raw.csv"
    with open(dst + "_kernels.json", "w") as fh:
        json.dump(kernels(rep), fh, indent=1)


if __name__ == "__main__":
    main()
