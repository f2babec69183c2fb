cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ for T in 1 0; do echo "GRAD_TG=$T"; GPK_GRAD_TGRAM=$T timeout 120 python tools/grad_timing.py; done; } > gpurun_out/t8.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
