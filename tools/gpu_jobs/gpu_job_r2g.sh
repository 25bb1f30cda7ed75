# round 2, job g: phase traces of the Cholesky kernel and the CPQR engine (debug stamps)
for nc in "4096 110" "262144 64" "8192 128" "4096 25"; do timeout 120 python tools/chol_trace.py $nc; done > gpurun_out/chol_trace_r2g.txt 2>&1
for ln in "110 4096" "64 16384" "272 8192" "25 800"; do timeout 120 python tools/engine_trace.py $ln; done > gpurun_out/engine_trace_r2g.txt 2>&1
echo done
