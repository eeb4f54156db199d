"""Top SASS lines of a kernel by a column of ncu's source page (e.g. stalls, shared-memory excess wavefronts)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
cols = sys.argv[3].split(",") if len(sys.argv) > 3 else ["Warp Stall Sampling (All Samples)"]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
key = cols[0]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(num(d[ix[key]]) for d in data if len(d) > ix[key])
print(f"total {key}: {tot:.0f}")
for d in sorted(data, key=lambda d: -num(d[ix[key]]) if len(d) > ix[key] else 0)[:top]:
    print(f"{d[ix['Address']]:>6s} " + " ".join(f"{num(d[ix[c]]):>10.0f}" for c in cols) + f"  {d[ix['Source']][:90]}")
