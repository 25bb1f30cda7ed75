# round 2, job h: traces after the compact Cholesky; GEMM fixed-cost probe; C2 bench; GPU suite
for nc in "4096 110" "262144 64" "8192 128"; do timeout 120 python tools/chol_trace.py $nc; done > gpurun_out/chol_trace_r2h.txt 2>&1
for c in 112 64 32; do timeout 300 python tools/gemm_overhead.py $c; done > gpurun_out/gemm_overhead_r2h.txt 2>&1
timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_r2h_c2.json 2> gpurun_out/bench_r2h_c2.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r2h_c4.json 2> gpurun_out/bench_r2h_c4.err
timeout 1700 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_r2h.log 2>&1; echo pytest_rc=$?
echo done
