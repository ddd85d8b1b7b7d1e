"""DRAM traffic per launch of the sweep kernel from an ncu --set full capture, for bench.py's
roofline.traffic (profiles/r02_traffic_<config>.json).

usage: python tools/ncu_traffic.py gpurun_out/x.ncu-rep cfg3 "<the command that was profiled>"
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, config, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head = rows[0]
col = {name: i for i, name in enumerate(head)}
launches = []
for r in rows[2:]:  # row 1 holds the units
    if len(r) < len(head) or "dag2_kernel" not in r[col["Kernel Name"]]:
        continue

    def num(key):
        return float(r[col[key]].replace(",", "")) if key in col and r[col[key]] else None

    launches.append({"dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
                     "duration_ns": num("gpu__time_duration.sum"),
                     "tensor_pipe_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                     "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")})
if not launches:
    sys.exit("no dag2_kernel launch in " + rep)
units = {"dram_read": 1.0, "dram_write": 1.0}
unit_row = rows[1]
for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    u = unit_row[col[key]].strip().lower()
    scale = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1.0)
    units["dram_read" if "read" in key else "dram_write"] = scale
l0 = launches[0]
rd, wr = l0["dram_read"] * units["dram_read"], l0["dram_write"] * units["dram_write"]
tu = unit_row[col["gpu__time_duration.sum"]].strip().lower()
to_ms = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(tu, 1.0)
res = {"kernel": "dag2_kernel", "config": config, "bytes_per_launch": int(rd + wr), "dram_read": int(rd),
       "dram_write": int(wr), "duration_ms_cold": l0["duration_ns"] * to_ms if l0["duration_ns"] else None,
       "tensor_pipe_pct": l0["tensor_pipe_pct"], "fp64_pipe_pct": l0["fp64_pipe_pct"],
       "source": f"ncu --set full --clock-control none (cold cache, one launch): {cmd}".strip()}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    f"r02_traffic_{config}.json")
json.dump(res, open(path, "w"), indent=1)
print(json.dumps(res))
