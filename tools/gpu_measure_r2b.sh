# Round-2 final measurement pass (session 3): GPU parity suite with the max-abs / rel-L2 report,
# the bench line, the ncu launch list of one bench step, one full ncu capture of a layer's
# kernels at 4465 tokens, one of the skinny lm_head GEMM at one row, and the attention comparators.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
PARITY_REPORT=gpurun_out/parity.json timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 300 gpurun_out/bench.json
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|attn|rms" --launch-skip 2600 --launch-count 2600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --skip-goodput --skip-live --skip-cpu > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gemm|attn" -s 5 -c 5 -o gpurun_out/layer_full_r2b python tools/prof_task.py --len 4465 --layers 2 --reps 1 > gpurun_out/ncu_full.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 2 -c 1 -o gpurun_out/skinny_lmhead_full python tools/skinny_ab.py --ops lm_head --ms 1 --iters 3 > gpurun_out/ncu_skinny.log 2>&1
timeout -s KILL 600 python tools/attn_compare.py --len 4465 --len 16384 > gpurun_out/attn_compare.log 2>&1
ls -la gpurun_out
