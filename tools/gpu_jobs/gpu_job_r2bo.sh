# round 2, job bo: final dress rehearsal after the epilogue change -- whole -m gpu suite, smoke, all bench lines, launch lists
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r2bo.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bo.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2bo.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r2bo.log
bash tools/refresh_profiles_r02.sh bench
bash tools/refresh_profiles_r02.sh launches
timeout 600 python bench.py --workload c4 --shard-of 8 --no-e2e > gpurun_out/shard_c4_of8_final2.json 2> gpurun_out/shard_c4_of8_final2.err
echo done
