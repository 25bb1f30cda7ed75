# round 2, job ad: GEMM parity incl. the two-CTA cases, then the round-2 bench lines
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gemm" > gpurun_out/pytest_r2ad.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2ad.log
bash tools/refresh_profiles_r02.sh bench
