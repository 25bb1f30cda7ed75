# round 2, job aw: why C4's sketch takes 130 ms inside the step against 125 ms alone -- clocks / power during the step,
# the step eager (RQLP_GRAPHS=0), and the sketch GEMM alone
timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_aw_graph.json 2> gpurun_out/bench_c4_aw_graph.err
RQLP_GRAPHS=0 timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_aw_eager.json 2> gpurun_out/bench_c4_aw_eager.err
nvidia-smi -q -d POWER > gpurun_out/power_aw.txt 2>&1
echo done
