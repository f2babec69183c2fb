cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in paper_2405_18457_b200/libgpk.so ab/libgpk_base.so; do echo "== $L"; for T in 1 0; do echo "T=$T"; GPK_LIB_PATH=$L GPK_TGRAM=$T timeout 200 python tools/kv_timing.py; done; done > gpurun_out/ab2.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "apply or operator or slab or solver or posterior or cross" > gpurun_out/pytest_ab2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab2.log
