#!/bin/bash
# ncu --set full of C2's three top kernels (first A-pass GEMM, CPQR engine, Cholesky) and of
# C1's first A-pass; summaries + per-kernel DRAM traffic under gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for k in gemm_tma hh_engine chol_blk; do
  RQLP_GRAPHS=0 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/ncu_c2_$k -f \
    python tools/run_one.py --workload c2 --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_c2_$k.ncu-rep > gpurun_out/ncu_c2_$k.txt
done
RQLP_GRAPHS=0 ncu --set full --clock-control none -k regex:gemm_tma -c 1 -o gpurun_out/ncu_c1_gemm_tma -f \
  python tools/run_one.py --workload c1 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_c1_gemm_tma.ncu-rep > gpurun_out/ncu_c1_gemm_tma.txt
echo done
