# round 2, job bf: engine (columns in global memory) with the register-column loops sized to the rows left:
# C5-shaped 1056 x 16384 B and other global-memory shapes, CPQR / tqlp parity, C5w bench
TAG=sized4 timeout 600 python tools/engine_bench.py 1056 16384 600 16384 528 32768 > gpurun_out/engine_sized4_r2bf.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cpqr or tqlp or tail" > gpurun_out/pytest_r2bf.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bf.log
timeout 900 python bench.py --workload c5w --no-e2e --no-cpu-baseline > gpurun_out/bench_c5w_bf.json 2> gpurun_out/bench_c5w_bf.err
echo done
