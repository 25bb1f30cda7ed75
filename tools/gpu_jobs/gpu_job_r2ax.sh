# round 2, job ax: C4's sketch (power-capped inside the step: 131 ms against 125 ms alone) as column slabs of other widths
for w in 0 64 96 128 112 80; do
  RQLP_NN_SLAB=$w timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_slab$w.json 2> gpurun_out/bench_c4_slab$w.err
done
echo done
