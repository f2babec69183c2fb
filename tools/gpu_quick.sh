cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 300 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |FAILED|passed|failed" | cut -c1-200 | head; timeout 300 python tools/config_smoke.py C1 C3 --steps 3 | cut -c1-600; } > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
