cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 120 python tools/ap_timing.py; GPK_AP_UPDATE=0 timeout 120 python tools/ap_timing.py; timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -2; timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200; } > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
