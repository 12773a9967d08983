set -x
timeout 600 python tools/attn_stamps.py --len 4465 > gpurun_out/attn_stamps.log 2>&1
timeout 900 python tools/attn_compare.py --len 4465 --len 16384 > gpurun_out/attn_compare.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem2sm tools/sanitizer/tmem2sm_repro.cu
for v in 0 1 2; do timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool racecheck /tmp/tmem2sm $v > gpurun_out/race_tmem2sm_v$v.log 2>&1; done
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_ops.py -q -x -k "forced_split and 300-1024-4096-1-5" > gpurun_out/race_pair.log 2>&1
timeout 600 python tools/prof_task.py --len 42 --len 163 --len 386 --len 872 --len 4465 --profile > gpurun_out/prof_short.log 2>&1
timeout 900 python bench.py --tp 1 --steps 2 --warmup 1 --tp-requests 8 > gpurun_out/bench_tp1.json 2> gpurun_out/bench_tp1.err
ls gpurun_out
