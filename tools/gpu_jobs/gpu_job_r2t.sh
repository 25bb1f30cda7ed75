# round 2, job t: non-polling warps spin on a shared flag instead of a barrier
run() { env "$@" TAG="$*" timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800; }
{ for m in 0 1 0 1; do run RQLP_ENGINE_SPIN=$m; done; } > gpurun_out/engine_ab_r2t.txt 2>&1
for m in 0 1; do RQLP_ENGINE_SPIN=$m RQLP_ENGINE_TRACE=2 timeout 120 python tools/engine_cta_trace.py 110 4096; done > gpurun_out/engine_cta_r2t.txt 2>&1
echo done
