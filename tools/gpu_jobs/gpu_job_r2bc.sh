# round 2, job bc: BRQLP W = orth(Z) as a span; the whole -m gpu suite on the final code, smoke, then the round's bench lines
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r2bc.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bc.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2bc.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r2bc.log
bash tools/refresh_profiles_r02.sh bench
echo done
