cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for F in 8 16 32 64; do echo "F=$F"; GPK_SGD_FLUSH=$F timeout 300 python tools/sgd_check.py 2>&1 | tail -2; done > gpurun_out/flush_sweep.log 2>&1
