nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/mma_rate tools/probes/mma_rate.cu && /tmp/mma_rate > gpurun_out/mma_rate.log 2>&1
cat gpurun_out/mma_rate.log
