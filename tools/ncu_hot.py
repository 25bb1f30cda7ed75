"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv` (SASS view)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
kern = None
rows = []
hdr = None
for line in out:
    if line.startswith('"Kernel Name"'):
        kern = line
        hdr = None
        continue
    if hdr is None:
        hdr = next(csv.reader([line]))
        continue
    if kfilter and kfilter not in (kern or ""):
        continue
    r = next(csv.reader([line]))
    d = dict(zip(hdr, r))
    try:
        rows.append((int(d["Warp Stall Sampling (All Samples)"]), d["Source"].strip(), d.get("Instructions Executed", "")))
    except (KeyError, ValueError):
        pass
tot = sum(x[0] for x in rows) or 1
print("total samples", tot)
for s, src, ie in sorted(rows, key=lambda t: -t[0])[:top]:
    print(f"{100 * s / tot:5.1f}%  {ie:>8}  {src[:100]}")
