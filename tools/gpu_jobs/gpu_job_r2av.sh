# round 2, job av: the optimistic row-sharded path (no per-orth readback) -- sharded tests, then the per-rank
# C4 block of an 8-rank run eager-optimistic, with graph replay (RQLP_SHARDED_GRAPHS=1) and careful (the old path)
timeout 1200 python -m pytest tests/test_dist_gpu.py tests/test_loopback_gpu.py tests/test_gpu_stress.py -x -q -p no:cacheprovider > gpurun_out/pytest_r2av.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2av.log
timeout 600 python bench.py --workload c4 --shard-of 8 --no-e2e > gpurun_out/shard_c4_of8_opt.json 2> gpurun_out/shard_c4_of8_opt.err
RQLP_SHARDED_GRAPHS=1 timeout 600 python bench.py --workload c4 --shard-of 8 --no-e2e > gpurun_out/shard_c4_of8_optgraph.json 2> gpurun_out/shard_c4_of8_optgraph.err
RQLP_SHARDED_OPTIMISTIC=0 timeout 600 python bench.py --workload c4 --shard-of 8 --no-e2e > gpurun_out/shard_c4_of8_careful.json 2> gpurun_out/shard_c4_of8_careful.err
timeout 600 python bench.py --workload c4 --shard-of 4 --no-e2e > gpurun_out/shard_c4_of4_opt.json 2> gpurun_out/shard_c4_of4_opt.err
timeout 600 python bench.py --workload c4 --shard-of 2 --no-e2e > gpurun_out/shard_c4_of2_opt.json 2> gpurun_out/shard_c4_of2_opt.err
echo done
