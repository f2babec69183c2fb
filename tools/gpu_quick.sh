cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 400 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |FAILED|passed|failed" | cut -c1-200 | head; timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200; GPK_GRAPHS=0 timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200; } > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log | tail -12
