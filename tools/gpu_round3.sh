cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/ffma2_bench > gpurun_out/ffma2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
GPK_KERNEL=1 timeout 300 python tools/kv_timing.py > gpurun_out/kv_timing_tc.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
