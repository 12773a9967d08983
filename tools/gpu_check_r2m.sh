for env in "" "FP_NARROW=0" "FP_SPLIT_OV_SCALE=0.5" "FP_SPLIT_OV_SCALE=0.25" "FP_STREAMK=0"; do
  echo "== env: $env"
  env $env timeout -s KILL 300 python tools/task_time.py --len 42 --len 163 --len 386 --len 545 --len 872 --len 1572 --reps 5 2>&1 | grep -v Warn
done > gpurun_out/task_time_env.log 2>&1
cat gpurun_out/task_time_env.log
