cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
GPK_DEVICE_POOL=0 timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_nopool.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_nopool.log
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_pool.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_pool.log
GPK_PHASE_TIMING=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_phase.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_phase.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
