# round 2, job bq: ncu --set full of the 64-wide block passes (NN and TN, two CTAs per SM) on the round's final binary
timeout 300 python tools/gemm_bench.py --reps 1 --shapes 262144,16384,64 > gpurun_out/ncu_gemm64_plain_bq.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -s 1 -c 3 -o gpurun_out/ncu_gemm64_r2bq python tools/gemm_bench.py --reps 1 --shapes 262144,16384,64 > gpurun_out/ncu_gemm64_r2bq.log 2>&1
echo done
