cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
GPK_SPD_INVERSE=0 GPK_PHASE_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/phase0.log 2>&1
grep '^{"set_hyper' gpurun_out/phase0.log | tail -2
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_r14.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
