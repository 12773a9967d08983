# compute-sanitizer pass of round 2 (logs under gpurun_out/, summaries in profiles/r2_sanitizer_*):
# racecheck on the attention kernel and the single-CTA split-K GEMM, synccheck on attention /
# split-K / stream-K, memcheck on smoke() and the attention ops, and racecheck on the 2-SM TMEM
# allocator reproducer (the pair GEMMs' only racecheck report).
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_ops.py -q -x -k "attn_prefill" > gpurun_out/race_attn.log 2>&1
timeout -s KILL 900 $CS --tool racecheck python -m pytest tests/test_gpu_ops.py -q -x -k "forced_split and 42-4096-4096" > gpurun_out/race_split_small.log 2>&1
timeout -s KILL 900 $CS --tool synccheck python -m pytest tests/test_gpu_ops.py -q -x -k "attn_prefill or forced_split or streamk" > gpurun_out/sync_ops.log 2>&1
timeout -s KILL 600 $CS --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.log 2>&1
timeout -s KILL 600 $CS --tool memcheck python -m pytest tests/test_gpu_ops.py -q -x -k attn > gpurun_out/memcheck_attn.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem2sm tools/sanitizer/tmem2sm_repro.cu
for v in 0 1 2; do timeout -s KILL 300 $CS --tool racecheck /tmp/tmem2sm $v > gpurun_out/race_tmem2sm_v$v.log 2>&1; done
for f in gpurun_out/race_*.log gpurun_out/sync_ops.log gpurun_out/memcheck_*.log; do echo "== $f"; tail -n 2 "$f"; done
