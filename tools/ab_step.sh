#!/bin/bash
# A/B of the device-timed bench step (no profiling events): base build (FP_AB_LIB) vs this
# build, ABBA order per round. Usage: tools/ab_step.sh <base.so> [rounds]
BASE=$1; R=${2:-2}
for i in $(seq 1 $R); do
  echo -n "base "; FP_AB_LIB=$BASE timeout 300 python tools/step_time.py | grep STEP_MS
  echo -n "new  "; timeout 300 python tools/step_time.py | grep STEP_MS
  echo -n "new  "; timeout 300 python tools/step_time.py | grep STEP_MS
  echo -n "base "; FP_AB_LIB=$BASE timeout 300 python tools/step_time.py | grep STEP_MS
done
