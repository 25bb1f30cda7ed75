# round 2, job k: engine A/B (record-first publish), PDL launch gap, ncu source view of the engine
for rf in 0 1; do RQLP_ENGINE_RECFIRST=$rf TAG=recfirst=$rf timeout 300 python tools/engine_bench.py 110 4096 64 16384 272 8192 25 800; done > gpurun_out/engine_ab_r2k.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pdl_gap tools/microbench/pdl_gap.cu && /tmp/pdl_gap > gpurun_out/pdl_gap_r2k.txt 2>&1
timeout 120 python tools/ncu_engine.py 110 4096 110 110 > gpurun_out/ncu_engine_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hh_engine -s 2 -c 2 -o gpurun_out/ncu_engine_r2k python tools/ncu_engine.py 110 4096 110 110 > gpurun_out/ncu_engine_r2k.log 2>&1
echo done
