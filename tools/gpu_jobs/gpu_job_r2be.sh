# round 2, job be: per-rank times of the strong-scaling runs and the C2 / C4 launch lists on the final code
for n in 2 4 8; do
  timeout 600 python bench.py --workload c4 --shard-of $n --no-e2e > gpurun_out/shard_c4_of${n}_final.json 2> gpurun_out/shard_c4_of${n}_final.err
done
RQLP_SHARDED_GRAPHS=1 timeout 600 python bench.py --workload c4 --shard-of 8 --no-e2e > gpurun_out/shard_c4_of8_final_graph.json 2> gpurun_out/shard_c4_of8_final_graph.err
timeout 600 python bench.py --workload c4 --shard-of 8 --shard-plain --no-e2e > gpurun_out/shard_c4_of8_final_plain.json 2> gpurun_out/shard_c4_of8_final_plain.err
timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_final_t1.json 2> gpurun_out/bench_c4_final_t1.err
bash tools/refresh_profiles_r02.sh launches
echo done
