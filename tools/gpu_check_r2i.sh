timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "attn" > gpurun_out/pytest_attn.log 2>&1; tail -3 gpurun_out/pytest_attn.log
timeout 600 python -m pytest tests/test_gpu_forward.py -q -x > gpurun_out/pytest_fwd.log 2>&1; tail -3 gpurun_out/pytest_fwd.log
bash tools/attn_variants.sh "w16:" "w16e3:-DFP_ATTN_EMU=3" "w16e4:-DFP_ATTN_EMU=4" > gpurun_out/attn_variants.log 2>&1
grep -v "^+" gpurun_out/attn_variants.log
