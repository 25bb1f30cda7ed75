# round 2, job bs: the whole -m gpu suite and smoke on the round's last commit
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r2bs.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bs.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2bs.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r2bs.log
timeout 900 python bench.py > gpurun_out/bench_c4_bs.json 2> gpurun_out/bench_c4_bs.err; echo rc=$? >> gpurun_out/bench_c4_bs.err
echo done
