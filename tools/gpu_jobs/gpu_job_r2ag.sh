# round 2, job ag: lazy (panel) updates of global-memory columns in the CPQR engine
{ for v in "RQLP_ENGINE_LAZY=0 RQLP_ENGINE_GLOBAL_THREADS=384" "RQLP_ENGINE_LAZY=1 RQLP_ENGINE_GLOBAL_THREADS=384" "RQLP_ENGINE_LAZY=0 RQLP_ENGINE_GLOBAL_THREADS=256" "RQLP_ENGINE_LAZY=1 RQLP_ENGINE_GLOBAL_THREADS=256"; do env $v TAG="$v" timeout 300 python tools/engine_bench.py 1056 16384 600 16384 600 8000; done; } > gpurun_out/engine_lazy_r2ag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cpqr or tqlp or qlp_tail or end_to_end" > gpurun_out/pytest_r2ag.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2ag.log
echo done
