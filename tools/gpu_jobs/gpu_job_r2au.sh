# round 2, job au: C5 at its own size (1048576 x 16384) on one B200, staged check against the oracle
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True timeout 2400 python tools/c5_full_check.py > gpurun_out/c5_full_1gpu_check.log 2>&1; echo rc=$? >> gpurun_out/c5_full_1gpu_check.log
echo done
