cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ for T in 1 0; do echo "T=$T"; GPK_TGRAM=$T timeout 120 python tools/ap_timing.py; GPK_TGRAM=$T GPK_AP_PROF=1 timeout 120 python tools/ap_timing.py; done; } > gpurun_out/t5.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 120 python tools/kv_timing.py 16384 26 65 >> gpurun_out/t5.log 2>&1
timeout 120 python tools/kv_timing.py 43008 20 65 >> gpurun_out/t5.log 2>&1
