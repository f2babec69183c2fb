cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 120 python tools/tg_check.py; } > gpurun_out/tg_check.log 2>&1
for T in 1 0; do for D in 0 2; do echo "T=$T D=$D"; GPK_TGRAM=$T GPK_KV_DBG=$D timeout 100 python tools/kv_timing.py 16384 26 65; done; done > gpurun_out/dbg.log 2>&1
for T in 1 0; do echo "T=$T"; GPK_TGRAM=$T GPK_TGRAM_MIN_D=3 timeout 200 python tools/kv_timing.py; done >> gpurun_out/dbg.log 2>&1
