cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for A in 1 0; do echo "AX=$A"; GPK_GRAD_AX=$A timeout 300 python tools/step_events.py 2>/dev/null | grep -E "grad_tc_kernel"; done > gpurun_out/t14.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/c2_20_gpu.py > gpurun_out/c2_20_gpu.log 2>&1
