# round 2, job e: C2 bench; ncu source-level captures of C2's Cholesky and CPQR engine kernels
set -x
timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_r2e_c2.json 2> gpurun_out/bench_r2e_c2.err
timeout 300 python tools/run_one.py --workload c2 --reps 2 > gpurun_out/r2e_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_blk_kernel -c 1 -o gpurun_out/ncu_r2e_chol -f python tools/run_one.py --workload c2 --reps 2 > gpurun_out/ncu_r2e_chol.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hh_engine_kernel -c 1 -o gpurun_out/ncu_r2e_engine -f python tools/run_one.py --workload c2 --reps 2 > gpurun_out/ncu_r2e_engine.log 2>&1
echo done
