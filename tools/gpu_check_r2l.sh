python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, os.getcwd())
from paper_2602_16603_b200 import build as B
subprocess.run(["nvcc", *B.NVCC_FLAGS, "-DFP_GEMM_STAMPS", "-o", "/tmp/gstamps.so", *B.sources()], check=True, capture_output=True)
PY
FP_AB_LIB=/tmp/gstamps.so FP_GEMM_STAMPS=1 timeout -s KILL 300 python tools/gemm_stamps.py 42,4096,4096,-1,0 42,6144,4096,-1,0 42,4096,14336,-1,0 42,28672,4096,-1,0 386,4096,4096,-1,0 872,6144,4096,-1,0 > gpurun_out/gemm_stamps.log 2>&1
cat gpurun_out/gemm_stamps.log
