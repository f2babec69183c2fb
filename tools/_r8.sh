cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
GPK_SGD_DBG=7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_slab -s 20 -c 1 -o gpurun_out/full_sgd_dbg7 -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_dbg7.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_slab -s 20 -c 1 -o gpurun_out/full_sgd_lazy7 -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_lazy7.log 2>&1
