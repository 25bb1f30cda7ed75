# round 2, job n: engine with the record first / warp-0-free poller; globaltimer cross-CTA trace
run() { env "$@" TAG="$*" timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800; }
{ run RQLP_ENGINE_W0FREE=0; run RQLP_ENGINE_W0FREE=1; } > gpurun_out/engine_ab_r2n.txt 2>&1
for w in 0 1; do RQLP_ENGINE_W0FREE=$w RQLP_ENGINE_TRACE=2 timeout 120 python tools/engine_cta_trace.py 110 4096; RQLP_ENGINE_W0FREE=$w timeout 120 python tools/engine_cta_trace.py 110 4096; done > gpurun_out/engine_cta_r2n.txt 2>&1
echo done
