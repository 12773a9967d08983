set -x
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/mma_rate tools/probes/mma_rate.cu && /tmp/mma_rate > gpurun_out/mma_rate.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:attn_prefill -s 2 -c 1 -o gpurun_out/attn_r2_base python tools/attn_compare.py --ours-only --len 4465 --reps 1 > gpurun_out/ncu_attn.log 2>&1
cat gpurun_out/mma_rate.log
