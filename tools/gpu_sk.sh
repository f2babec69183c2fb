cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 500 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | cut -c1-300 | head -20
  for V in 1 0; do echo "== GPK_KV_STREAMK=$V"; GPK_KV_STREAMK=$V timeout 200 python tools/kv_timing.py 2>&1 | cut -c1-200
  GPK_KV_STREAMK=$V timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200; done; } > gpurun_out/sk.log 2>&1
cat gpurun_out/sk.log
