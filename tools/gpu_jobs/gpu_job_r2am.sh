# round 2, job am: C2-sized A-pass as 64 + 48 at two CTAs per SM vs one 112-wide tile
{ for v in "X=0" "RQLP_GEMM_SPLIT_NARROW=1" "RQLP_GEMM_SPLIT_NARROW=1 RQLP_GEMM_OCC2_FORCE=1" "RQLP_GEMM_OCC2_FORCE=1"; do echo "$v"; env $v timeout 300 python tools/gemm_bench.py --reps 20 --shapes 4096,4096,110 4096,4096,64 4096,4096,48 2000,2000,125; done; } > gpurun_out/gemm_c2_r2am.txt 2>&1
for v in "X=0" "RQLP_GEMM_SPLIT_NARROW=1 RQLP_GEMM_OCC2_FORCE=1"; do env $v timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > "gpurun_out/bench_c2_am_$(echo $v | tr -d ' =')".json 2>/dev/null; done
echo done
