# round 2, job at: per-rank times behind the projected strong scaling (one rank's row block of an N-GPU run through the
# sharded NCCL handle at world size 1, and the same block on the single-GPU graph-replay handle), and C5 at its own
# size (1048576 x 16384, 137 GB) on ONE B200
for n in 2 4 8; do
  timeout 600 python bench.py --workload c4 --shard-of $n --no-e2e > gpurun_out/shard_c4_of${n}_nccl.json 2> gpurun_out/shard_c4_of${n}_nccl.err
  timeout 600 python bench.py --workload c4 --shard-of $n --shard-plain --no-e2e > gpurun_out/shard_c4_of${n}_plain.json 2> gpurun_out/shard_c4_of${n}_plain.err
done
timeout 900 python bench.py --workload c5 --shard-of 8 --no-e2e > gpurun_out/shard_c5_of8_nccl.json 2> gpurun_out/shard_c5_of8_nccl.err
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 1500 python bench.py --workload c5 --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_c5_full_1gpu.json 2> gpurun_out/bench_c5_full_1gpu.err; echo rc=$? >> gpurun_out/bench_c5_full_1gpu.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/bench_c5_full_1gpu.err
echo done
