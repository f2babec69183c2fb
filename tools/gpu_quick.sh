cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -2; GPK_PHASE_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep set_hyper | tail -2; timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200; } > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
