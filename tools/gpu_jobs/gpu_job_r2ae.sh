# round 2, job ae: C5-shaped engine (1056 x 16384, columns in global memory): step time along j
timeout 300 python tools/engine_trace_steps.py 1056 16384 > gpurun_out/engine_steps_r2ae.txt 2>&1
timeout 300 python tools/engine_bench.py 1056 16384 > gpurun_out/engine_bench_c5_r2ae.txt 2>&1
echo done
