cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 200 python tools/kv_timing.py; GPK_KV_DEEP=1 timeout 200 python tools/kv_timing.py;
  timeout 200 python tools/sgd_timing.py 393216 1; GPK_KV_DEEP=1 timeout 200 python tools/sgd_timing.py 393216 1;
  GPK_KV_DEEP=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2; } > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log | cut -c1-330
