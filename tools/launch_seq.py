import csv, sys
path, nper = sys.argv[1], int(sys.argv[2])
rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
ours = [r for r in rows if "rqlpk" in r["Kernel Name"]][-nper:]
for r in ours:
    name = r["Kernel Name"].split("(")[0].replace("rqlpk::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    t = float(r["Metric Value"]); u = r["Metric Unit"]
    t = t / 1000.0 if u in ("ns", "nsecond") else (t * 1000.0 if u in ("ms", "msecond") else t)
    print(f"{t:8.1f}  {name}  grid={r.get('Grid Size','')}")
