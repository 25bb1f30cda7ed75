# round 2, job az: per-launch list (grid sizes, times) of one eager C4 factorisation, to look at the small products
# of the block orthonormalisation / deflation (the b_other stage, 33 ms)
RQLP_GRAPHS=0 timeout 600 python tools/run_one.py --workload c4 --reps 2 > gpurun_out/run_c4_az.log 2>&1 && \
RQLP_GRAPHS=0 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4_az.csv python tools/run_one.py --workload c4 --reps 2 > /dev/null 2>&1
echo done
