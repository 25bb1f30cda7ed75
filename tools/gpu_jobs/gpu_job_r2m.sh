# round 2, job m: engine exchange variants (record spacing, candidate copies, warp-0-free poller)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/microbench/latency.cu && /tmp/lat > gpurun_out/latency_r2m.txt 2>&1
run() { env "$@" TAG="$*" timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800; }
{
run RQLP_ENGINE_RSTRIDE=4 RQLP_ENGINE_NCOPY=1
run RQLP_ENGINE_RSTRIDE=2 RQLP_ENGINE_NCOPY=1
run RQLP_ENGINE_RSTRIDE=8 RQLP_ENGINE_NCOPY=1
run RQLP_ENGINE_RSTRIDE=16 RQLP_ENGINE_NCOPY=1
run RQLP_ENGINE_RSTRIDE=8 RQLP_ENGINE_NCOPY=4
run RQLP_ENGINE_RSTRIDE=8 RQLP_ENGINE_NCOPY=8
run RQLP_ENGINE_RSTRIDE=16 RQLP_ENGINE_NCOPY=8
run RQLP_ENGINE_RSTRIDE=8 RQLP_ENGINE_NCOPY=4 RQLP_ENGINE_W0FREE=1
run RQLP_ENGINE_RSTRIDE=16 RQLP_ENGINE_NCOPY=8 RQLP_ENGINE_W0FREE=1
} > gpurun_out/engine_ab_r2m.txt 2>&1
for v in "RQLP_ENGINE_RSTRIDE=8 RQLP_ENGINE_NCOPY=4" "RQLP_ENGINE_RSTRIDE=16 RQLP_ENGINE_NCOPY=8 RQLP_ENGINE_W0FREE=1"; do env $v timeout 120 python tools/engine_cta_trace.py 110 4096; done > gpurun_out/engine_cta_r2m.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cpqr or qlp_tail or end_to_end or brqlp or tqlp or ties" -p no:cacheprovider > gpurun_out/pytest_r2m.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2m.log
echo done
