"""Per-kernel DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) from an ncu report ->
profiles/ncu_traffic.json (read by bench.py for the roofline 'traffic' field)."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
res = {}
for d in data:
    name = d[ix["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[ix[k]]) * scale.get(units[ix[k]], 1)
    t = float(d[ix["gpu__time_duration.sum"]]) * (1e-3 if units[ix["gpu__time_duration.sum"]] == "us" else 1)
    f64 = float(d[ix["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]]) \
        if "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active" in ix else None
    res.setdefault(name, []).append({"dram_bytes": b, "ms": t, "fp64": f64})
summary = {k: {"dram_bytes_per_launch": sum(x["dram_bytes"] for x in v) / len(v),
               "ms_per_launch_ncu": sum(x["ms"] for x in v) / len(v), "launches_captured": len(v),
               "fp64_pipe_pct": v[0]["fp64"]}
           for k, v in res.items()}
summary["_source"] = rep
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
