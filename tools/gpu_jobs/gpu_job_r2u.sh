# round 2, job u: A-pass DMMA efficiency per tile width (C4-sized A)
timeout 900 python tools/gemm_bench.py --reps 8 --shapes 262144,16384,48 262144,16384,64 262144,16384,80 262144,16384,96 262144,16384,112 262144,16384,128 262144,16384,144 262144,16384,528 > gpurun_out/gemm_bn_r2u.txt 2>&1
echo done
