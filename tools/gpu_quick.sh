cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 120 python tools/ap_timing.py; GPK_FUSED_AP=0 timeout 120 python tools/ap_timing.py; timeout 200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "solver or ap" 2>&1 | tail -3; } > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
