cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "solvers or apply_columns or optimise" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_tc.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
python tools/kv_timing.py 16384 26 65 > gpurun_out/kv_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kv_tc -s 2 -c 1 -o gpurun_out/kv_tc_c2 \
    python tools/kv_timing.py 16384 26 65 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kv_tc -s 30 -c 1 -o gpurun_out/kv_tc_apslab \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_ap.log 2>&1
echo "ncu full ap rc=$?" >> gpurun_out/ncu_full_ap.log
