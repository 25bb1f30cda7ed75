# round 2, job z: ncu source view of the Cholesky kernel (C2's 110 x 110), fine sampling
timeout 120 python tools/orth_bench.py --reps 4 --shapes 4096,110 > gpurun_out/ncu_chol_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_blk -s 2 -c 4 -o gpurun_out/ncu_chol_r2z python tools/orth_bench.py --reps 4 --shapes 4096,110 > gpurun_out/ncu_chol_r2z.log 2>&1
echo done
