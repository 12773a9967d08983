timeout -s KILL 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_forward.py tests/test_gpu_tp.py tests/test_gpu_moe.py -q -x > gpurun_out/pytest_attn.log 2>&1; tail -2 gpurun_out/pytest_attn.log
timeout -s KILL 300 python tools/attn_stamps.py --len 4465 > gpurun_out/attn_stamps.log 2>&1; tail -9 gpurun_out/attn_stamps.log
timeout -s KILL 300 python tools/attn_compare.py --ours-only --len 4465 --len 16384 2>&1 | grep TFLOP
timeout -s KILL 300 python tools/task_time.py --len 42 --len 163 --len 386 --len 545 --len 872 --len 1572 --len 4465 --reps 5 2>&1 | grep "M="
