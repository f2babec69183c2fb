cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
GPK_TGRAM_MIN_D=3 timeout 900 python -m pytest tests -m gpu -q -x -k "apply or operator or slab or solver or posterior or cross" > gpurun_out/pytest_gpu_tg3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_tg3.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
