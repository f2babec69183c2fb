cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ python tools/timeline.py 3 2>&1 | grep -v Warn | head -14
  GPK_AUX_PRIORITY=0 python tools/timeline.py 3 2>&1 | grep -v Warn | head -3
  GPK_AP_PROF=1 timeout 120 python tools/ap_timing.py 2>&1 | tail -3
  timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200
  GPK_AUX_PRIORITY=0 timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200; } > gpurun_out/tl.log 2>&1
cat gpurun_out/tl.log
