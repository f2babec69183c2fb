cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
GPK_AP_PROF=1 timeout 120 python tools/ap_timing.py > gpurun_out/approf.log 2>&1
timeout 120 python tools/ap_timing.py >> gpurun_out/approf.log 2>&1
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_pool.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_pool.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
