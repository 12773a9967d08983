python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, os.getcwd())
from paper_2602_16603_b200 import build as B
subprocess.run(["nvcc", *B.NVCC_FLAGS, "-DFP_GEMM_STAMPS", "-o", "/tmp/stamps.so", *B.sources()], check=True, capture_output=True)
PY
FP_STAMPS_LIB=/tmp/stamps.so CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/attn_stamps.py --len 4465 --reps 1 > gpurun_out/stamps_dbg.log 2>&1; echo "stamps rc=$?" >> gpurun_out/stamps_dbg.log
FP_STAMPS_LIB=/tmp/stamps.so timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tools/attn_stamps.py --len 1000 --reps 1 > gpurun_out/stamps_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/stamps_memcheck.log
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_ops.py -q -x -k attn > gpurun_out/attn_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/attn_synccheck.log
tail -5 gpurun_out/stamps_dbg.log gpurun_out/stamps_memcheck.log gpurun_out/attn_synccheck.log
