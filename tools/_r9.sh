cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TEST_TIMEOUT=1500 bash tools/gpu_run.sh tests
TAG=c4 bash tools/gpu_run.sh bench
timeout 300 python tools/one_step.py C4 1 > gpurun_out/one_step_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file gpurun_out/launches_c4.csv python tools/one_step.py C4 1 > gpurun_out/launches_ncu.log 2>&1
timeout 2700 python tools/make_golden_scale.py c5 > gpurun_out/golden_c5.log 2>&1; echo "rc=$?" >> gpurun_out/golden_c5.log
