# round 2, job s: engine exchange reads as atomics (home L2 slice) vs relaxed loads
run() { env "$@" TAG="$*" timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800; }
{ for m in 0 1 2 3 0; do run RQLP_ENGINE_ATOMPOLL=$m; done; } > gpurun_out/engine_ab_r2s.txt 2>&1
for m in 0 1 3; do RQLP_ENGINE_ATOMPOLL=$m RQLP_ENGINE_TRACE=2 timeout 120 python tools/engine_cta_trace.py 110 4096; done > gpurun_out/engine_cta_r2s.txt 2>&1
echo done
