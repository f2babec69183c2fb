cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/sgd_check.py > gpurun_out/sgd_check.log 2>&1; echo "rc=$?" >> gpurun_out/sgd_check.log
GPK_SGD_GRAM=0 timeout 300 python tools/sgd_check.py > gpurun_out/sgd_check_nogram.log 2>&1
if grep -q "C4 epoch" gpurun_out/sgd_check.log; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_slab -s 20 -c 1 -o gpurun_out/full_sgd_lazy3 -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_lazy3.log 2>&1
fi
