# round 2, job f: GPU suite (+ stress tests), C2 / C3 / C4 benches
set -x
timeout 1700 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider --durations=15 > gpurun_out/pytest_r2f.log 2>&1; echo pytest_rc=$?
for w in c2 c3 c4; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/bench_r2f_$w.json 2> gpurun_out/bench_r2f_$w.err; done
echo done
