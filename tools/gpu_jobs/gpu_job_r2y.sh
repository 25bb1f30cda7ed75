# round 2, job y: BRQLP ||A||^2 on the last narrow block's A W pass instead of the sketch
for f in 0 1; do RQLP_FRO_LATE=$f timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_frolate$f.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_loopback_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2y.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2y.log
echo done
