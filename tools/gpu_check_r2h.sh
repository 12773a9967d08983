bash tools/attn_variants.sh "emu3:" "emu2:-DFP_ATTN_EMU=2" "emu4:-DFP_ATTN_EMU=4" "emu5:-DFP_ATTN_EMU=5" "emu0:-DFP_ATTN_EMU=0" > gpurun_out/attn_variants.log 2>&1
grep -v "^+" gpurun_out/attn_variants.log
