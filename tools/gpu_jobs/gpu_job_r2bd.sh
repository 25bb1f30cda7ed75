# round 2, job bd: the full-size C4 factorisation against the oracle again, on the final code (span-only bases,
# transposed E product) -- ~17 min of host CPU for the oracle
timeout 3000 python tools/full_parity.py --workload c4 --out gpurun_out/r02_c4_full_parity.json > gpurun_out/r02_c4_full_parity.log 2>&1; echo rc=$? >> gpurun_out/r02_c4_full_parity.log
echo done
