"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals of the LAST factorisation."""
import collections
import csv
import sys

path = sys.argv[1]
nper = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
ours = [r for r in rows if "rqlpk" in r["Kernel Name"]]
half = ours[-nper:] if nper else ours[len(ours) // 2:]
agg = collections.OrderedDict()
for r in half:
    name = r["Kernel Name"].split("(")[0].replace("rqlpk::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    t = float(r["Metric Value"])
    u = r["Metric Unit"]
    t = t / 1000.0 if u in ("ns", "nsecond") else (t * 1000.0 if u in ("ms", "msecond") else t)
    agg.setdefault(name, [0.0, 0])
    agg[name][0] += t
    agg[name][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"{'us':>10} {'share':>6} {'n':>4}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{v[0]:10.1f} {100 * v[0] / tot:5.1f}% {v[1]:4d}  {k[:80]}")
print(f"{tot:10.1f}  total us over {len(half)} launches")
