#!/bin/bash
# A/B of the device-timed bench step between two environment settings of THIS build, ABBA
# order. Usage: tools/ab_env.sh "<env A>" "<env B>" [rounds]   e.g. tools/ab_env.sh "FP_NARROW=0" "" 2
A=$1; B=$2; R=${3:-2}
for i in $(seq 1 $R); do
  echo -n "A "; env $A timeout 300 python tools/step_time.py | grep STEP_MS
  echo -n "B "; env $B timeout 300 python tools/step_time.py | grep STEP_MS
  echo -n "B "; env $B timeout 300 python tools/step_time.py | grep STEP_MS
  echo -n "A "; env $A timeout 300 python tools/step_time.py | grep STEP_MS
done
