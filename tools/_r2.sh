cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/sgd_check.py > gpurun_out/sgd_check.log 2>&1; echo "rc=$?" >> gpurun_out/sgd_check.log
if grep -q "C4 epoch" gpurun_out/sgd_check.log; then
  TEST_TIMEOUT=900 bash tools/gpu_run.sh tests
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_slab -s 20 -c 1 -o gpurun_out/full_sgd_lazy -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_lazy.log 2>&1
  timeout 900 python tools/make_golden_scale.py c4 > gpurun_out/golden_c4.log 2>&1; echo "rc=$?" >> gpurun_out/golden_c4.log
fi
