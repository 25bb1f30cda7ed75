# round 2, job aj: ||A||^2 streamed beside the plain sketch pass (two streams) vs the 96-wide split
for v in 1 0 1 0; do RQLP_FRO_SPLIT96=$v timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_split96_$v.json 2>/dev/null; done
for v in 1 0; do RQLP_FRO_SPLIT96=$v timeout 600 python bench.py --workload c3 --steps 6 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_split96_$v.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_loopback_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2aj.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2aj.log
echo done
