#!/bin/bash
# A/B per-kernel timing of the bench's 16 request lengths: base library (FP_AB_LIB) vs this build
# on the same box, in ABBA order per round (GPU clocks drift under the power cap, so a fixed
# order would bias the comparison). Usage: tools/ab_prof.sh <base.so> [rounds]
BASE=$1; R=${2:-1}
L="--len 4465 --len 163 --len 3971 --len 545 --len 386 --len 3997 --len 1572 --len 504 --len 42 --len 438 --len 451 --len 1021 --len 872 --len 437 --len 5389 --len 853"
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  FP_AB_LIB=$BASE timeout 300 python tools/prof_task.py --profile $L > gpurun_out/prof_base${i}a.txt 2>&1
  timeout 300 python tools/prof_task.py --profile $L > gpurun_out/prof_new${i}a.txt 2>&1
  timeout 300 python tools/prof_task.py --profile $L > gpurun_out/prof_new${i}b.txt 2>&1
  FP_AB_LIB=$BASE timeout 300 python tools/prof_task.py --profile $L > gpurun_out/prof_base${i}b.txt 2>&1
done
