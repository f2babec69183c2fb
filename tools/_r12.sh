cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/sgd_check.py > gpurun_out/sgd_check.log 2>&1
TEST_TIMEOUT=1800 bash tools/gpu_run.sh tests
timeout 900 python tools/config_smoke.py C1 C2 C3 --steps 3 > gpurun_out/configs.log 2>&1
