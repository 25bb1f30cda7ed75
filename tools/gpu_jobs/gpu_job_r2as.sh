# round 2, job as: re-entry validation of HEAD — full -m gpu suite, smoke, the default bench line (C4) and C2
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_r2as.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r2as.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2as.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2as.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r2as.log
timeout 900 python bench.py > gpurun_out/bench_c4_r2as.json 2> gpurun_out/bench_c4_r2as.err; echo rc=$? >> gpurun_out/bench_c4_r2as.err
timeout 300 python bench.py --workload c2 > gpurun_out/bench_c2_r2as.json 2> gpurun_out/bench_c2_r2as.err
echo done
