# round 2, job bn: the direct alpha/beta epilogue (tiles <= 64 wide) loads a row's old C values together before
# combining and storing them (they were 32 dependent round trips per thread)
timeout 600 python tools/gemm_bench.py --reps 20 --shapes 262144,16384,64 > gpurun_out/gemm_bn.txt 2>&1
for rep in 1 2; do
  timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_bn_$rep.json 2>> gpurun_out/bench_c4_bn.err
done
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_fullsize.py tests/test_gpu_stress.py tests/test_loopback_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_r2bn.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bn.log
echo done
