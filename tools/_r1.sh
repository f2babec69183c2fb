cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_run.sh tests
timeout 200 python tools/tf32_peak.py > gpurun_out/tf32.log 2>&1
TAG=c4 bash tools/gpu_run.sh bench
timeout 300 python tools/one_step.py C4 1 > gpurun_out/one_step_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file gpurun_out/launches_c4.csv python tools/one_step.py C4 1 > gpurun_out/launches_ncu.log 2>&1
timeout 200 python tools/sgd_timing.py 393216 1 > gpurun_out/sgd_timing.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_tc_kernel -s 20 -c 1 -o gpurun_out/full_sgd_slab -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_slab.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_update_pack -s 20 -c 1 -o gpurun_out/full_sgd_update -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_upd.log 2>&1
echo done
