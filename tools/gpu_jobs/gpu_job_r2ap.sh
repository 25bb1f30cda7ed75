# round 2, job ap: CPQR engine CTA count (the all-to-all exchange costs 3660 cycles at 148 CTAs, 2820 at 74)
{ for g in 148 111 74 56 37 148; do RQLP_ENGINE_G=$g TAG="G<=$g" timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800 1056 16384; done; } > gpurun_out/engine_g_r2ap.txt 2>&1
echo done
