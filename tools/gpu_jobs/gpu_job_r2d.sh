# round 2, job d: GPU suite after block CGS2 + the ||A||^2 warp; C4 (fused vs separate ||A||^2), C2
set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_r2d.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r2d_c4.json 2> gpurun_out/bench_r2d_c4.err
RQLP_FRO_FUSED=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r2d_c4_fro0.json 2> gpurun_out/bench_r2d_c4_fro0.err
timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_r2d_c2.json 2> gpurun_out/bench_r2d_c2.err
RQLP_FRO_FUSED=0 timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_r2d_c2_fro0.json 2> gpurun_out/bench_r2d_c2_fro0.err
timeout 600 python bench.py --workload c5w --no-cpu-baseline --no-e2e > gpurun_out/bench_r2d_c5w.json 2> gpurun_out/bench_r2d_c5w.err
echo done
