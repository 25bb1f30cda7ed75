# round 2, job bg: dress rehearsal of the round-end checks on the final code -- the whole -m gpu suite, smoke,
# then every bench line again (engine change: c5w, c3) and the launch lists
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r2bg.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bg.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2bg.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r2bg.log
bash tools/refresh_profiles_r02.sh bench
bash tools/refresh_profiles_r02.sh launches
echo done
