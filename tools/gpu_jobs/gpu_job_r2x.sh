# round 2, job x: two CTAs per SM for the narrow widths (16..48) too; streamed BRQLP host outputs
for o in 0 64 0 64; do echo "RQLP_GEMM_OCC2=$o"; RQLP_GEMM_OCC2=$o timeout 600 python tools/gemm_bench.py --reps 8 --shapes 262144,16384,16 262144,16384,32 262144,16384,48 4096,110,110 4096,4096,32 65536,272,272; done > gpurun_out/gemm_occ_r2x.txt 2>&1
for o in 0 64; do RQLP_GEMM_OCC2=$o timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_occ_r2x_$o.json 2>/dev/null; RQLP_GEMM_OCC2=$o timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_occ_r2x_$o.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2x.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2x.log
echo done
