# round 2, job q: critical-path warp = the highest warp index (scheduler priority) in the engine and the Cholesky
run() { env "$@" TAG="$*" timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800 110 110 64 64; }
{ run RQLP_ENGINE_CRIT=0; run RQLP_ENGINE_CRIT=1; run RQLP_ENGINE_CRIT=0; run RQLP_ENGINE_CRIT=1; } > gpurun_out/engine_ab_r2q.txt 2>&1
{ for lw in 0 1 0 1; do echo "RQLP_CHOL_LW=$lw"; RQLP_CHOL_LW=$lw timeout 300 python tools/orth_bench.py --shapes 4096,110 262144,64 110,110 8192,128; done; } > gpurun_out/orth_ab_r2q.txt 2>&1
for lw in 0 1; do RQLP_CHOL_LW=$lw timeout 120 python tools/chol_trace.py 4096 110; done > gpurun_out/chol_trace_r2q.txt 2>&1
for v in "RQLP_ENGINE_CRIT=0 RQLP_CHOL_LW=0" "RQLP_ENGINE_CRIT=1 RQLP_CHOL_LW=1"; do env $v timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_$(echo $v | tr -d ' =').json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2q.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2q.log
echo done
