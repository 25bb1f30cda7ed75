# round 2, job ay: C4's sketch as 3 x 128 + 144 columns (RQLP_COLSPLIT_PREFER=128, now the default) against 3 x 144 + 96
for rep in 1 2; do for w in 144 128; do
  RQLP_COLSPLIT_PREFER=$w timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_prefer${w}_$rep.json 2> gpurun_out/bench_c4_prefer${w}_$rep.err
done; done
for w in 144 128; do RQLP_COLSPLIT_PREFER=$w timeout 600 python bench.py --workload c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_prefer${w}.json 2> gpurun_out/bench_c3_prefer${w}.err; done
echo done
