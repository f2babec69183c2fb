cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/grad_timing.py 16384 26 64 > gpurun_out/grad_sanity.log 2>&1 || { echo "sanity rc=$?" >> gpurun_out/grad_sanity.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/grad_timing.py > gpurun_out/grad_timing.log 2>&1; echo "rc=$?" >> gpurun_out/grad_timing.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"kv_reduce_dot|grad_tc_kernel" -s 20 -c 2 \
    -o gpurun_out/r10_reduce_grad python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
