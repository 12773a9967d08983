#!/bin/bash
# A/B of two library builds on the same box, interleaved: A = the committed HEAD (built from
# `git archive` into the snapshot's tools/_ab_prev, prepared on the CPU side), B = the working
# tree's in-tree build. Usage: bash tools/ab_lib.sh <prev_lib.so> [rounds]
PREV=$1; R=${2:-2}
for i in $(seq 1 $R); do
  for v in A B; do
    if [ $v = A ]; then export FP_AB_LIB=$PREV; else unset FP_AB_LIB; fi
    echo "== $v round $i"
    timeout -s KILL 200 python tools/attn_compare.py --ours-only --len 4465 --len 16384 --reps 5 2>&1 | grep TFLOP
    timeout -s KILL 200 python tools/task_time.py --len 386 --len 1572 --len 4465 --reps 3 2>&1 | grep "M="
  done
done
