PARITY_REPORT=gpurun_out/parity.json timeout -s KILL 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python tools/attn_stamps.py --len 4465 > gpurun_out/attn_stamps.log 2>&1; tail -12 gpurun_out/attn_stamps.log
