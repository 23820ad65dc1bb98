"""Summarise ncu output into small tracked JSON files under profiles/.

    python tools/ncu_summary.py full   <report.ncu-rep> <out.json>
    python tools/ncu_summary.py launch <launches.csv>   <out.json>

`full`: per captured launch, the metrics that back the design choices (pipe
utilisation, DRAM bytes, occupancy, issue activity).  `launch`: per kernel name,
launch count, total and mean device time and share of the total (from a
`--metrics gpu__time_duration.sum` run; cold-cache, serialised: compare shares).
"""
import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    launches = []
    for d in data:
        rec = {"kernel": d[idx["Kernel Name"]]}
        for m in FULL_METRICS:
            if m in idx:
                v = d[idx[m]].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                rec[m + (f" [{units[idx[m]]}]" if units[idx[m]] else "")] = v
        launches.append(rec)
    json.dump({"source": rep, "launches": launches}, open(out, "w"), indent=1)


def launch(csv_path, out):
    lines = [ln for ln in open(csv_path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"]
        a = agg.setdefault(k, {"launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += float(r["Metric Value"].replace(",", "")) / (1e3 if r["Metric Unit"] == "ns" else 1)
    tot = sum(a["total_us"] for a in agg.values())
    res = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]):
        res.append({"kernel": k, **a, "mean_us": a["total_us"] / a["launches"], "share": a["total_us"] / tot})
    json.dump({"source": csv_path, "total_us": tot, "kernels": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    {"full": full, "launch": launch}[sys.argv[1]](sys.argv[2], sys.argv[3])
