cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/ap_timing.py > gpurun_out/ap_timing.log 2>&1 || { echo "ap rc=$?" >> gpurun_out/ap_timing.log; exit 1; }
GPK_FUSED_AP=0 timeout 120 python tools/ap_timing.py >> gpurun_out/ap_timing.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_r15.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
