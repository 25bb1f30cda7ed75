# round 2, job ar: one-CTA thread-per-column CPQR for short wide B (C1's 25 x 800) vs the grid engine
{ for v in 0 1 0 1; do RQLP_ENGINE_CTA=$v TAG="cta=$v" timeout 300 python tools/engine_bench.py 25 800 16 1000 20 600 26 800; done; } > gpurun_out/engine_cta_r2ar.txt 2>&1
for v in 0 1; do for w in c1 c1e; do RQLP_ENGINE_CTA=$v timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_${w}_cta$v.json 2>/dev/null; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_r2ar.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2ar.log
echo done
