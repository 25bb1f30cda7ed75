# round 2, job r: GEMM producer thread in warp 0 vs the last consumer warp
for pw in 0 7 0 7; do echo "RQLP_GEMM_PRODUCER_WARP=$pw"; RQLP_GEMM_PRODUCER_WARP=$pw timeout 600 python tools/gemm_bench.py --reps 10 --shapes 262144,16384,64 4096,4096,110 65536,8192,272 262144,16384,16; done > gpurun_out/gemm_ab_r2r.txt 2>&1
echo done
