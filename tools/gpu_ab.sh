# A/B of the working tree's libgpk.so against ab/libgpk_base.so (another build
# of the same C-ABI, via GPK_LIB_PATH): operator timing, AP solve, C2 bench.
# usage (under gpurun): bash tools/gpu_ab.sh [tests]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ if [ "$1" = tests ]; then timeout 400 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "^E  |FAILED|passed|failed|Error" | cut -c1-300 | head -20; fi
  for L in paper_2405_18457_b200/libgpk.so ${LIBS:-ab/libgpk_base.so}; do
    echo "== $L"
    GPK_LIB_PATH=$L timeout 200 python tools/kv_timing.py 2>&1 | cut -c1-260
    GPK_LIB_PATH=$L timeout 120 python tools/ap_timing.py 2>&1 | tail -1
    GPK_LIB_PATH=$L timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200
  done; } > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
