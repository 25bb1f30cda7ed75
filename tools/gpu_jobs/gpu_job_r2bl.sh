# round 2, job bl: L2 prefetch of the C tile for the direct beta epilogue (BRQLP's X -= V_<j C products)
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_fullsize.py tests/test_gpu_stress.py tests/test_loopback_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_r2bl.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bl.log
for rep in 1 2; do
  timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_bl_$rep.json 2>> gpurun_out/bench_c4_bl.err
done
timeout 600 python tools/gemm_bench.py --reps 20 --shapes 262144,16384,64 262144,16384,528 > gpurun_out/gemm_bl.txt 2>&1
echo done
