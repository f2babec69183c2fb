cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 200 python tools/sgd_timing.py 393216 1; timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -2; timeout 300 python tools/config_smoke.py C4 C1 C3 --steps 2; } > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log | cut -c1-700
