# round 2, job an: two-CTA threshold in (tile, k-tile) units (the m x 64 Grams now run in gram64)
{ for u in 40000 10000 40000 10000; do echo "RQLP_GEMM_OCC2_UNITS=$u"; RQLP_GEMM_OCC2_UNITS=$u timeout 300 python tools/gemm_bench.py --reps 10 --shapes 262144,64,64 262144,128,64 262144,256,64 262144,384,64 16384,512,64; done; } > gpurun_out/gemm_units_r2an.txt 2>&1
for u in 40000 10000; do RQLP_GEMM_OCC2_UNITS=$u timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_units$u.json 2>/dev/null; done
echo done
