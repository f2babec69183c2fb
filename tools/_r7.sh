cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for D in 0 4 7; do echo "DBG=$D"; GPK_SGD_DBG=$D timeout 300 python tools/sgd_check.py 2>&1 | tail -2; done > gpurun_out/dbg_sweep.log 2>&1
timeout 300 python tools/sgd_check.py > gpurun_out/sgd_check.log 2>&1
