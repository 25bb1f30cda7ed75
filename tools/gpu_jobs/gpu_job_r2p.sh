# round 2, job p: engine record slot spacing (old 3-word format) and poll back-off
run() { env "$@" TAG="$*" timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800; }
{ run RQLP_ENGINE_RSTRIDE=4; run RQLP_ENGINE_RSTRIDE=16; run RQLP_ENGINE_BACKOFF=50; run RQLP_ENGINE_BACKOFF=200; run RQLP_ENGINE_RSTRIDE=16 RQLP_ENGINE_BACKOFF=100; run RQLP_ENGINE_RSTRIDE=4; } > gpurun_out/engine_ab_r2p.txt 2>&1
echo done
