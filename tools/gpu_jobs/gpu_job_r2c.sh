# round 2, job c: GPU suite, C4 bench (fused vs separate ||A||^2), C2/C3/C5w benches, C4 launch list
set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_r2c.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r2c_c4.json 2> gpurun_out/bench_r2c_c4.err
RQLP_FRO_FUSED=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r2c_c4_fro0.json 2> gpurun_out/bench_r2c_c4_fro0.err
for w in c2 c3 c5w; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_r2c_$w.json 2> gpurun_out/bench_r2c_$w.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2c_c4.csv python tools/run_one.py --workload c4 --reps 1 > gpurun_out/ncu_r2c_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -c 16 -o gpurun_out/ncu_r2c_c4_gemm -f python tools/run_one.py --workload c4 --reps 1 > gpurun_out/ncu_r2c_full.log 2>&1
echo done
