# round 2, job j: engine phase trace + stage timing baseline; Cholesky trace
for ln in "110 4096" "64 16384" "272 8192" "25 800" "110 110"; do timeout 120 python tools/engine_trace.py $ln; done > gpurun_out/engine_trace_r2j.txt 2>&1
timeout 300 python tools/engine_bench.py > gpurun_out/engine_bench_r2j.txt 2>&1
for nc in "4096 110" "262144 64"; do timeout 120 python tools/chol_trace.py $nc; done > gpurun_out/chol_trace_r2j.txt 2>&1
echo done
