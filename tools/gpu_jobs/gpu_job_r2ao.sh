# round 2, job ao: cross-SM exchange latency microbenchmark (the engine's record exchange alone)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exchange tools/microbench/exchange.cu && timeout 120 /tmp/exchange > gpurun_out/exchange_r2ao.txt 2>&1
echo done
