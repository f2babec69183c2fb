cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 120 python tools/tg_check.py; GPK_TGRAM=0 timeout 120 python tools/tg_check.py; } > gpurun_out/tg_check.log 2>&1
for T in 1 0; do GPK_TGRAM=$T timeout 200 python tools/kv_timing.py >> gpurun_out/tg_timing.log 2>&1; echo "T=$T rc=$?" >> gpurun_out/tg_timing.log; done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
