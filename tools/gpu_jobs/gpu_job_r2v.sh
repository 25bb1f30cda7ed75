# round 2, job v: 64-wide GEMM with 2 CTAs per SM (3-stage rings) vs 1
for o in 0 1 0 1; do echo "RQLP_GEMM_OCC2=$o"; RQLP_GEMM_OCC2=$o timeout 600 python tools/gemm_bench.py --reps 8 --shapes 262144,16384,64 262144,64,64 262144,512,64 16384,512,64; done > gpurun_out/gemm_occ_r2v.txt 2>&1
for o in 0 1; do RQLP_GEMM_OCC2=$o timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_occ$o.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2v.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2v.log
echo done
