set -x
bash tools/attn_variants.sh "base:" "st4:-DFP_ATTN_STAGES=4" "st4tree:-DFP_ATTN_STAGES=4 -DFP_ATTN_TREE_MAX" "st5:-DFP_ATTN_STAGES=5" > gpurun_out/attn_variants.log 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_ops.py -q -x -k "forced_split and 1-5-300-1024-4096" > gpurun_out/race_pair.log 2>&1
tail -3 gpurun_out/race_pair.log
