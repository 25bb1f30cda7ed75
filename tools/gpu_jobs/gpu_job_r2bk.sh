# round 2, job bk: the short-K 64-wide NN product without the beta epilogue (plain gemm_nn), K = 64 .. 1024, to
# separate the read-modify-write epilogue from the K-loop in BRQLP's X -= V_<j C products (450 us at K = 384 with beta = 1)
timeout 600 python tools/gemm_bench.py --reps 20 --shapes 262144,64,64 262144,128,64 262144,384,64 262144,512,64 262144,1024,64 262144,4096,64 > gpurun_out/gemm_shortk_r2bk.txt 2>&1
echo done
