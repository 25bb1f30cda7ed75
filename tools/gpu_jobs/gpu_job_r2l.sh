# round 2, job l: per-CTA engine trace; ncu source view of the grid engine (110 x 4096)
for rf in 1 0; do for ln in "110 4096" "64 16384"; do RQLP_ENGINE_RECFIRST=$rf timeout 120 python tools/engine_cta_trace.py $ln; done; done > gpurun_out/engine_cta_r2l.txt 2>&1
timeout 120 python tools/ncu_engine.py 110 4096 > gpurun_out/ncu_engine_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hh_engine -s 1 -c 1 -o gpurun_out/ncu_engine_grid_r2l python tools/ncu_engine.py 110 4096 > gpurun_out/ncu_engine_r2l.log 2>&1
echo done
