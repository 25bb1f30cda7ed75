#!/bin/bash
# Regenerate the measured artifacts under gpurun_out/ (copied to profiles/ by hand):
# bench lines per workload, the C2 launch list (ncu, serialized), the paper tables.
set -u
cd "$(dirname "$0")/.."
python paper_1811_09334_b200/build.py > /dev/null 2>&1
python -c "import oracle; oracle.build()"
mkdir -p gpurun_out
for w in c1 c1e c2; do   # the defaults (20 timed steps, 5 warm-up)
  python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.log
done
python bench.py --workload c3 --steps 10 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log
python bench.py --workload c5w --steps 3 --warmup 5 > gpurun_out/bench_c5w.json 2> gpurun_out/bench_c5w.log
RQLP_GRAPHS=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python tools/run_one.py --workload c2 --reps 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_c2.csv "$(python tools/run_one.py --workload c2 --reps 1 | awk '{print $3}')" \
  > gpurun_out/launches_c2.txt
python tools/paper_tables.py --out gpurun_out/paper_tables.json > gpurun_out/paper_tables.md 2> gpurun_out/paper_tables.log
echo done
