# round 2, job bi: whole-tile runs for the short-K 64-wide NN products (gemm_tma_kernel WT variant)
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_fullsize.py tests/test_gpu_stress.py -x -q -p no:cacheprovider > gpurun_out/pytest_r2bi.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bi.log
for v in 1 0 1 0; do
  RQLP_GEMM_WT=$v timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_wt${v}_$RANDOM.json 2>> gpurun_out/bench_c4_wt.err
done
RQLP_GEMM_WT=1 timeout 600 python bench.py --workload c5w --no-e2e --no-cpu-baseline > gpurun_out/bench_c5w_wt1.json 2>> gpurun_out/bench_c4_wt.err
RQLP_GEMM_WT=1 timeout 600 python bench.py --workload c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_wt1.json 2>> gpurun_out/bench_c4_wt.err
echo done
