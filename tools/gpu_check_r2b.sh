set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
PARITY_REPORT=gpurun_out/parity.json timeout 1200 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --skip-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/attn_stamps.py --len 4465 > gpurun_out/attn_stamps.log 2>&1
timeout 900 python tools/attn_compare.py --len 4465 --len 16384 > gpurun_out/attn_compare.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem2sm tools/sanitizer/tmem2sm_repro.cu && timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool racecheck /tmp/tmem2sm > gpurun_out/race_tmem2sm.log 2>&1
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_ops.py -q -x -k "forced_split and 42-4096-4096" > gpurun_out/race_split_small.log 2>&1
tail -2 gpurun_out/*.log
