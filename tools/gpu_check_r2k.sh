bash tools/attn_timing.sh "r32_112:" "r40_104:-DFP_ATTN_REGS_CTRL=40 -DFP_ATTN_REGS_SOFTMAX=104" "stamps:-DFP_GEMM_STAMPS" > gpurun_out/attn_timing.log 2>&1
cat gpurun_out/attn_timing.log
