cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2405_18457_b200/libgpk.so ab/libgpk_c2d.so paper_2405_18457_b200/libgpk.so ab/libgpk_c2d.so; do echo "== $L"; GPK_LIB_PATH=$L timeout 120 python tools/ap_timing.py | cut -c1-200; GPK_LIB_PATH=$L GPK_AP_PROF=1 timeout 120 python tools/ap_timing.py 2>&1 | grep phases; done > gpurun_out/t11.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
