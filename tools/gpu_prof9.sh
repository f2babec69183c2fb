cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
GPK_PHASE_TIMING=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/phase9.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_v9.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ap_persistent -s 1 -c 1 -o gpurun_out/ap_full9 -f \
    python tools/ap_timing.py > gpurun_out/ncu_ap9.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_ap9.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_tc_kernel -s 2 -c 1 -o gpurun_out/kv_full9 -f \
    python tools/kv_timing.py 16384 26 65 > gpurun_out/ncu_kv9.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_kv9.log
