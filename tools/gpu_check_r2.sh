set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_ops.py -q -x -k "attn_prefill" > gpurun_out/race_attn.log 2>&1
timeout 900 $CS --tool racecheck python -m pytest tests/test_gpu_ops.py -q -x -k "forced_split or streamk" > gpurun_out/race_split.log 2>&1
timeout 900 $CS --tool synccheck python -m pytest tests/test_gpu_ops.py -q -x -k "attn_prefill or forced_split or streamk" > gpurun_out/sync_ops.log 2>&1
timeout 900 $CS --tool racecheck --target-processes all python -m pytest tests/test_gpu_tp_ipc.py tests/test_gpu_tp.py -q -x > gpurun_out/race_tp.log 2>&1
tail -3 gpurun_out/*.log
