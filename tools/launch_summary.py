"""Per-kernel totals / shares from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import sys
from collections import defaultdict

path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
tot, cnt = defaultdict(float), defaultdict(int)
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].replace("void ", "").split("(")[0]
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r["Metric Unit"], 1e-6)
    tot[name] += float(r["Metric Value"].replace(",", "")) * scale
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"# ncu launch list of `{cmd}` (gpu__time_duration.sum, --clock-control none; cold-cache serialised "
      "launches: compare shares)")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} launches {cnt[k]:4d}  total {tot[k]:8.3f} ms  share {100 * tot[k] / all_ms:5.1f}%  "
          f"per-launch {tot[k] / cnt[k]:.4f} ms")
