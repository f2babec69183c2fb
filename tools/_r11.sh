cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TEST_TIMEOUT=1800 bash tools/gpu_run.sh tests
timeout 900 python tools/config_smoke.py C1 C2 C3 C5 --steps 2 > gpurun_out/configs.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_slab -s 20 -c 1 -o gpurun_out/full_sgd_slab_r02 -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_slab_r02.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_apply -s 20 -c 1 -o gpurun_out/full_sgd_apply_r02 -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_apply_r02.log 2>&1
