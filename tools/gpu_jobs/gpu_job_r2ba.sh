# round 2, job ba: BRQLP E = V_j^T V_<j as the transposed c0 x b_j product, CholeskyQR2 of block_orth in place
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_loopback_gpu.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "brqlp or BRQLP or sweep or c4 or autorank or loopback" > gpurun_out/pytest_r2ba.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2ba.log
timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_ba.json 2> gpurun_out/bench_c4_ba.err
echo done
