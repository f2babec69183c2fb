cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/ex2_check > gpurun_out/t7.log 2>&1
for L in paper_2405_18457_b200/libgpk.so ab/libgpk_mufu.so; do echo "== $L"; GPK_LIB_PATH=$L timeout 120 python tools/ap_timing.py; GPK_LIB_PATH=$L GPK_AP_PROF=1 timeout 120 python tools/ap_timing.py 2>&1 | grep phases; GPK_LIB_PATH=$L timeout 120 python tools/kv_timing.py 16384 26 65; GPK_LIB_PATH=$L timeout 120 python tools/kv_timing.py 43008 20 65; done >> gpurun_out/t7.log 2>&1
