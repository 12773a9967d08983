bash tools/attn_timing.sh "base:" "split:-DFP_ATTN_SPLIT_P" "base2:" "split2:-DFP_ATTN_SPLIT_P" > gpurun_out/attn_timing.log 2>&1
cat gpurun_out/attn_timing.log
FP_AB_LIB=/tmp/fpt_split/libflowprefill.so timeout -s KILL 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_forward.py -q -x -k "attn or oracle or golden or preemption" 2>&1 | tail -2
for v in base split; do echo "== task $v"; FP_AB_LIB=/tmp/fpt_$v/libflowprefill.so timeout -s KILL 200 python tools/task_time.py --len 386 --len 1572 --len 4465 --reps 3 2>&1 | grep "M="; done
