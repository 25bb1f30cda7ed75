# round 2, job ac: ncu --set full of the 64-wide block pass (TN and NN, two CTAs per SM), C4-sized A
timeout 300 python tools/gemm_bench.py --reps 1 --shapes 262144,16384,64 > gpurun_out/ncu_gemm64_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -s 1 -c 3 -o gpurun_out/ncu_gemm64_r2ac python tools/gemm_bench.py --reps 1 --shapes 262144,16384,64 > gpurun_out/ncu_gemm64_r2ac.log 2>&1
echo done
