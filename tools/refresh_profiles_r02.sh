#!/bin/bash
# Round-2 measured artifacts under gpurun_out/ (copied to profiles/r02_* by hand):
#   part "bench": bench lines per workload (+ the reference arm on the default C4 workload)
#   part "launches": ncu launch lists (gpu__time_duration, serialised, cold) of one C2 and one C4
#   factorisation (eager: RQLP_GRAPHS=0), after the same command exited 0 without ncu
set -u
cd "$(dirname "$0")/.."
part=${1:-bench}
python paper_1811_09334_b200/build.py > /dev/null 2>&1
python -c "import oracle; oracle.build()"
mkdir -p gpurun_out
if [ "$part" = bench ]; then
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02_gpu.txt 2>&1
  lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/r02_host.txt 2>&1
  for w in c1 c1e c2; do
    timeout 600 python bench.py --workload $w > gpurun_out/r02_bench_$w.json 2> gpurun_out/r02_bench_$w.log
  done
  timeout 900 python bench.py --workload c3 --steps 10 --warmup 5 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.log
  timeout 1200 python bench.py --workload c5w --steps 3 --warmup 3 > gpurun_out/r02_bench_c5w.json 2> gpurun_out/r02_bench_c5w.log
  timeout 1200 python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.log
  timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_bench_reference_c4.json 2> gpurun_out/r02_bench_reference_c4.log
else
  for w in c2 c4; do
    RQLP_GRAPHS=0 timeout 600 python tools/run_one.py --workload $w --reps 2 > gpurun_out/r02_run_$w.log 2>&1 && \
    RQLP_GRAPHS=0 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r02_launches_$w.csv python tools/run_one.py --workload $w --reps 2 > /dev/null 2>&1
    n=$(awk '{print $3}' gpurun_out/r02_run_$w.log | tail -1)
    python tools/launch_table.py gpurun_out/r02_launches_$w.csv "$n" > gpurun_out/r02_launches_$w.txt
  done
fi
echo done
