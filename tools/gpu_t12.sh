cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 300 python tools/c1_compare.py; GPK_DENSE_CAP=0 timeout 300 python tools/c1_compare.py; } > gpurun_out/c1cmp.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
