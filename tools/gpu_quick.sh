cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/quick.log
GPK_PHASE_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/phase.log 2>&1
grep '^{"set_hyper' gpurun_out/phase.log | tail -2 >> gpurun_out/quick.log
timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-250 >> gpurun_out/quick.log
cat gpurun_out/quick.log
