# round 2, job ab: Cholesky with the tile warps off warp 0's sub-partition (per-tile loop)
{ for b in 0 2 0 2; do echo "RQLP_CHOL_BATCH=$b"; RQLP_CHOL_BATCH=$b timeout 300 python tools/orth_bench.py --shapes 4096,110 262144,64 110,110 8192,128 2000,125; done; } > gpurun_out/orth_batch_r2ab.txt 2>&1
for b in 0 2; do RQLP_CHOL_BATCH=$b timeout 120 python tools/chol_trace.py 4096 110; done > gpurun_out/chol_trace_r2ab.txt 2>&1
echo done
