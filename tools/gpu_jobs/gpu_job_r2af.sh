# round 2, job af: global-memory-column engine path with 256 / 384 / 512 threads (columns in flight)
{ for t in 256 384 512 256 384 512; do RQLP_ENGINE_GLOBAL_THREADS=$t TAG="threads=$t" timeout 300 python tools/engine_bench.py 1056 16384 600 16384 1056 4096; done; } > gpurun_out/engine_global_r2af.txt 2>&1
for t in 256 384; do RQLP_ENGINE_GLOBAL_THREADS=$t timeout 300 python tools/engine_trace_steps.py 1056 16384; done > gpurun_out/engine_steps_r2af.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cpqr or tqlp or qlp_tail" > gpurun_out/pytest_r2af.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2af.log
echo done
