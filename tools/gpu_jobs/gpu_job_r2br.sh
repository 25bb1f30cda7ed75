# round 2, job br: replica check of the summed B on the sharded path -- sharded tests, then the per-rank C4 block (8 ranks) and C4
timeout 1500 python -m pytest tests/test_loopback_gpu.py tests/test_dist_gpu.py tests/test_gpu_stress.py -x -q -p no:cacheprovider > gpurun_out/pytest_r2br.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2br.log
timeout 600 python bench.py --workload c4 --shard-of 8 --no-e2e > gpurun_out/shard_c4_of8_repcheck.json 2> gpurun_out/shard_c4_of8_repcheck.err
RQLP_REPLICA_CHECK=0 timeout 600 python bench.py --workload c4 --shard-of 8 --no-e2e > gpurun_out/shard_c4_of8_norepcheck.json 2> gpurun_out/shard_c4_of8_norepcheck.err
timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_br.json 2> gpurun_out/bench_c4_br.err
echo done
