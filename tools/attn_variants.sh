#!/bin/bash
# Build attention-kernel variants (compile-time macros) as separate copies of the library under
# /tmp and time each with tools/attn_compare.py --ours-only (FP_AB_LIB selects the copy), plus
# the phase stamps of each variant. Usage: bash tools/attn_variants.sh "name:-DFLAG ..." ...
set -u
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  out=/tmp/fpv_$name
  mkdir -p $out
  python - "$out" $flags <<'PY'
import os, subprocess, sys
sys.path.insert(0, os.getcwd())
from paper_2602_16603_b200 import build as B
out, flags = sys.argv[1], sys.argv[2:]
subprocess.run([os.environ.get("NVCC", "nvcc"), *B.NVCC_FLAGS, *flags, "-o", out + "/libflowprefill.so", *B.sources()], check=True, capture_output=True)
subprocess.run([os.environ.get("NVCC", "nvcc"), *B.NVCC_FLAGS, *flags, "-DFP_GEMM_STAMPS", "-o", out + "/libstamps.so", *B.sources()], check=True, capture_output=True)
PY
  echo "== variant $name ($flags)"
  FP_AB_LIB=$out/libflowprefill.so python tools/attn_compare.py --ours-only --len 4465 --len 16384 2>&1 | grep TFLOP
  FP_STAMPS_LIB=$out/libstamps.so python tools/attn_stamps.py --len 4465 2>&1 | grep -E "phases|MMA:|median" | head -4
done
