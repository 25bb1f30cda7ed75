# round 2, job ah: global-memory-column engine: 384 threads, L2 prefetch of the warp's next column
{ for v in 0 1 0 1; do RQLP_ENGINE_PREFETCH=$v TAG="prefetch=$v" timeout 300 python tools/engine_bench.py 1056 16384 600 16384 600 8000; done; } > gpurun_out/engine_pf_r2ah.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cpqr or tqlp or qlp_tail" > gpurun_out/pytest_r2ah.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2ah.log
echo done
