# round 2, job ai: the whole -m gpu suite and smoke() on the current code
timeout 2400 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/pytest_r2ai.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2ai.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2ai.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r2ai.log
echo done
