# round 2, job bj: C5 whole on one B200 again on the final code (engine loops sized to the rows left): staged check + bench line
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 2400 python tools/c5_full_check.py > gpurun_out/c5_full_1gpu_check.log 2>&1; echo rc=$? >> gpurun_out/c5_full_1gpu_check.log
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 1500 python bench.py --workload c5 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_c5_full_1gpu.json 2> gpurun_out/bench_c5_full_1gpu.err; echo rc=$? >> gpurun_out/bench_c5_full_1gpu.err
timeout 900 python bench.py --workload c5 --shard-of 8 --no-e2e > gpurun_out/shard_c5_of8_final.json 2> gpurun_out/shard_c5_of8_final.err
echo done
