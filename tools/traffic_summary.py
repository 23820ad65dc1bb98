"""Per-launch DRAM and L2 write traffic of the bench step's tensor-core conv launches from an
ncu --csv metrics log, as profiles/traffic_<workload>.json (the file bench.py's roofline
'traffic' field reads).  Usage:
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
lts__t_sectors_srcunit_tex_op_write.sum -k regex:tc_conv_kernel --csv --log-file L.csv \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-graph
  python tools/traffic_summary.py L.csv out.json <launches per step> <source note>"""
import collections
import csv
import io
import json
import sys

path, out, per_step = sys.argv[1], sys.argv[2], int(sys.argv[3])
note = sys.argv[4] if len(sys.argv) > 4 else ""
txt = open(path).read()
start = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
launch = collections.OrderedDict()
for r in rows:
    key = r["ID"]
    d = launch.setdefault(key, {"kernel": r["Kernel Name"][:90]})
    v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] not in ("", "n/a") else 0.0
    unit = r.get("Metric Unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024 ** 2, "GB": 1024 ** 3,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1)
    d[r["Metric Name"]] = v * scale
L = list(launch.values())
step = L[:per_step]  # the first step (the eager step bench.py runs before timing: same kernels and data)
res = {
    "source": note,
    "unit": "bytes per bench step's tensor-core conv launches (the unit the bench roofline's 'achieved' covers)",
    "dram_bytes_per_launch_unit": sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in step),
    "dram_read": sum(x.get("dram__bytes_read.sum", 0) for x in step),
    "dram_write": sum(x.get("dram__bytes_write.sum", 0) for x in step),
    "l2_write_bytes_from_sms": 32 * sum(x.get("lts__t_sectors_srcunit_tex_op_write.sum", 0) for x in step),
    "note": "DRAM writes of a launch undercount its outputs by what is still dirty in L2 when it ends; the L2 "
            "write bytes received from the SMs (32 B sectors) are the outputs as written - against the algorithmic "
            "output bytes they show whether stores are wasted",
    "per_launch": [{"kernel": x["kernel"], "read": x.get("dram__bytes_read.sum"), "write": x.get("dram__bytes_write.sum"),
                    "l2_write": 32 * x.get("lts__t_sectors_srcunit_tex_op_write.sum", 0),
                    "us": x.get("gpu__time_duration.sum")} for x in step],
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res)[:400])
