# round 2, job w: 2-CTA/SM rule (tiles >= 296 or tiles x ktiles >= 40000); C4 bench; full GPU suite
timeout 600 python tools/gemm_bench.py --reps 8 --shapes 262144,16384,64 262144,64,64 262144,512,64 16384,512,64 > gpurun_out/gemm_occ_r2w.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_r2w.json 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_r2w.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2w.log
echo done
