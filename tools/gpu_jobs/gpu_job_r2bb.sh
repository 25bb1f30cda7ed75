# round 2, job bb: BRQLP pre-power block orthonormalisation as span only (one projection + one CholeskyQR pass)
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_loopback_gpu.py tests/test_gpu_fullsize.py tests/test_dist_gpu.py tests/test_gpu_stress.py -x -q -p no:cacheprovider > gpurun_out/pytest_r2bb.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bb.log
timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_bb.json 2> gpurun_out/bench_c4_bb.err
RQLP_BRQLP_PRE_SPAN=0 timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_bb_off.json 2> gpurun_out/bench_c4_bb_off.err
echo done
