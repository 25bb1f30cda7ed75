#!/bin/bash
# Probe a GPU box: FP64 peaks (DFMA/DMMA), cuBLAS DGEMM reference, host cores, clocks.
mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g) > gpurun_out/host.txt 2>&1
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_probe.csv &
SMI=$!
./tools/microbench/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
python - > gpurun_out/dgemm_torch.txt 2>&1 << 'PY'
import torch, time
for (m,n,k) in [(8192,8192,8192),(65536,272,8192),(8192,272,65536),(4096,112,4096)]:
    a=torch.randn(m,k,dtype=torch.float64,device='cuda'); b=torch.randn(k,n,dtype=torch.float64,device='cuda')
    for _ in range(3): c=a@b
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): c=a@b
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/10
    print(m,n,k, "%.3f ms  %.2f TFLOP/s"%(ms, 2*m*n*k/ms/1e9))
PY
kill $SMI
