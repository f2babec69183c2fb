cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/grad_timing.py 16384 26 64 > gpurun_out/grad_sanity.log 2>&1 || { echo "sanity rc=$?" >> gpurun_out/grad_sanity.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/grad_timing.py > gpurun_out/grad_timing.log 2>&1; echo "rc=$?" >> gpurun_out/grad_timing.log
timeout 600 python tools/sgd_timing.py 393216 1 > gpurun_out/sgd_timing.log 2>&1; echo "rc=$?" >> gpurun_out/sgd_timing.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_r11.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
