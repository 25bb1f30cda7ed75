# round 2, job i (session 2 re-entry): state check of HEAD — full GPU suite, default bench (C4), C2 bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2i_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_r2i_c4.json 2> gpurun_out/bench_r2i_c4.err
timeout 300 python bench.py --workload c2 > gpurun_out/bench_r2i_c2.json 2> gpurun_out/bench_r2i_c2.err
timeout 2400 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_r2i.log 2>&1; echo pytest_rc=$?
echo done
