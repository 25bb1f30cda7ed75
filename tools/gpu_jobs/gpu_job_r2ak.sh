# round 2, job ak: dedicated m x <=64 Gram kernel (upper-triangle 8x8 tiles, one smem tile for both operands)
{ for v in 0 1 0 1; do echo "RQLP_GRAM64=$v"; RQLP_GRAM64=$v timeout 300 python tools/orth_bench.py --shapes 262144,64 131072,64 4096,64 100000,16 30000,40; done; } > gpurun_out/orth_gram_r2ak.txt 2>&1
for v in 0 1; do RQLP_GRAM64=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_gram$v.json 2>/dev/null; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_loopback_gpu.py tests/test_gpu_stress.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2ak.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2ak.log
echo done
