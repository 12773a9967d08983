timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "attn" > gpurun_out/pytest_attn.log 2>&1; tail -2 gpurun_out/pytest_attn.log
bash tools/attn_variants.sh "desc:" "desc_st4:-DFP_ATTN_STAGES=4" "desc_tree:-DFP_ATTN_TREE_MAX" > gpurun_out/attn_variants.log 2>&1
grep -v "^+" gpurun_out/attn_variants.log
