#!/bin/bash
# Build attention-kernel variants (compile-time macros) as separate library copies under /tmp and
# time each with tools/attn_compare.py --ours-only, every run under a hard 90 s kill.
#   bash tools/attn_timing.sh "name:-DFLAG ..." ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  out=/tmp/fpt_$name; mkdir -p $out
  python - "$out" $flags <<'PY'
import os, subprocess, sys
sys.path.insert(0, os.getcwd())
from paper_2602_16603_b200 import build as B
out, flags = sys.argv[1], sys.argv[2:]
r = subprocess.run([os.environ.get("NVCC", "nvcc"), *B.NVCC_FLAGS, *flags, "-o", out + "/libflowprefill.so", *B.sources()], capture_output=True, text=True)
log = r.stdout + r.stderr
i = log.find("attn_prefill_tc_kernel")
print("build rc", r.returncode, [l.strip() for l in log[i:i + 600].splitlines() if "spill" in l][:1])
PY
  echo "== $name ($flags)"
  FP_AB_LIB=$out/libflowprefill.so timeout -s KILL 90 python tools/attn_compare.py --ours-only --len 4465 --len 16384 --reps 5 2>&1 | grep -E "TFLOP|Error|error" ; echo "rc=${PIPESTATUS[0]}"
done
