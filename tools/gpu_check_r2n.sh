PARITY_REPORT=gpurun_out/parity.json timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_ops.py -q -x -k attn > gpurun_out/race_attn.log 2>&1; tail -2 gpurun_out/race_attn.log
timeout -s KILL 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.log 2>&1; tail -2 gpurun_out/memcheck_smoke.log
timeout -s KILL 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_ops.py -q -x -k attn > gpurun_out/memcheck_attn.log 2>&1; tail -2 gpurun_out/memcheck_attn.log
