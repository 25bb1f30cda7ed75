# round 2, job aa: Cholesky phase 3 in batches of 4 tiles per warp
{ for b in 0 1 0 1; do echo "RQLP_CHOL_BATCH=$b"; RQLP_CHOL_BATCH=$b timeout 300 python tools/orth_bench.py --shapes 4096,110 262144,64 110,110 8192,128 2000,125; done; } > gpurun_out/orth_batch_r2aa.txt 2>&1
for b in 0 1; do RQLP_CHOL_BATCH=$b timeout 120 python tools/chol_trace.py 4096 110; done > gpurun_out/chol_trace_r2aa.txt 2>&1
for b in 0 1; do RQLP_CHOL_BATCH=$b timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_batch$b.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2aa.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2aa.log
echo done
