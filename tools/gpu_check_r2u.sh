bash tools/attn_timing.sh "base:" "spec:-DFP_ATTN_SPEC_MAX" "base2:" "spec2:-DFP_ATTN_SPEC_MAX" > gpurun_out/attn_timing.log 2>&1
cat gpurun_out/attn_timing.log
FP_AB_LIB=/tmp/fpt_spec/libflowprefill.so timeout -s KILL 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_forward.py -q -x -k "attn or oracle or golden or preemption or batch" 2>&1 | tail -2
