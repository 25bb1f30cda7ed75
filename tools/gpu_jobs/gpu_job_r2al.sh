# round 2, job al: the dedicated Gram kernel up to 128 columns (C2's 110 x 110 Grams) vs 64
{ for v in 64 128 64 128; do echo "RQLP_GRAM_MAX=$v"; RQLP_GRAM_MAX=$v timeout 300 python tools/orth_bench.py --shapes 4096,110 2000,125 8192,128 65536,100 262144,64; done; } > gpurun_out/orth_gram_r2al.txt 2>&1
for v in 64 128 64 128; do RQLP_GRAM_MAX=$v timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram$v.json 2>/dev/null; cp gpurun_out/bench_c2_gram$v.json gpurun_out/bench_c2_gram${v}_$RANDOM.json; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2al.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2al.log
echo done
