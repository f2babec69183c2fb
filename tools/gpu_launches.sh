# Phase split (synchronising timer) + ncu launch list of a short C2 bench run.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
GPK_PHASE_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/phase.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_${1:-x}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
tail -5 gpurun_out/phase.log | cut -c1-600
