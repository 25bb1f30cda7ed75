set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_r2b.log 2>&1; echo pytest_rc=$?
for v in default FRO0 CS0; do
  case $v in default) E="";; FRO0) E="RQLP_FRO_FUSED=0";; CS0) E="RQLP_GEMM_COLSPLIT=0";; esac
  env $E timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r2b_$v.json 2> gpurun_out/bench_r2b_$v.err
done
timeout 600 python tools/gemm_bench.py --shapes 262144,16384,528 65536,8192,272 262144,16384,64 262144,16384,16 > gpurun_out/gemm_r2b.txt 2>&1
RQLP_GEMM_COLSPLIT=0 timeout 600 python tools/gemm_bench.py --shapes 262144,16384,528 65536,8192,272 > gpurun_out/gemm_r2b_cs0.txt 2>&1
