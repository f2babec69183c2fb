cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2405_18457_b200/libgpk.so ab/libgpk_st4.so paper_2405_18457_b200/libgpk.so ab/libgpk_st4.so; do echo "== $L"; GPK_LIB_PATH=$L timeout 120 python tools/ap_timing.py | cut -c1-120; GPK_LIB_PATH=$L GPK_AP_PROF=1 timeout 120 python tools/ap_timing.py 2>&1 | grep phases; done > gpurun_out/t13.log 2>&1
