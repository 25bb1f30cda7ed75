# round 2, job aq: lanes per shared-memory column group (8 / 16 / 32) for CTAs with <= 32 columns
{ for g in 8 16 32 8 16; do RQLP_ENGINE_GSM=$g TAG="gsm=$g" timeout 300 python tools/engine_bench.py 110 4096 25 800 64 4096 128 4096; done; } > gpurun_out/engine_gsm_r2aq.txt 2>&1
for g in 8 16; do RQLP_ENGINE_GSM=$g timeout 300 python bench.py --workload c2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gsm$g.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cpqr or qlp_tail or end_to_end or ties" > gpurun_out/pytest_r2aq.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2aq.log
RQLP_ENGINE_GSM=16 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "cpqr or qlp_tail or end_to_end or ties" > gpurun_out/pytest_r2aq16.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2aq16.log
echo done
