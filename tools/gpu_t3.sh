cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for L in paper_2405_18457_b200/libgpk.so ab/libgpk_base.so; do echo "== $L"; GPK_LIB_PATH=$L timeout 120 python tools/ap_timing.py; GPK_LIB_PATH=$L timeout 120 python tools/grad_timing.py; done > gpurun_out/t3.log 2>&1
echo "TG min 3" >> gpurun_out/t3.log; GPK_TGRAM_MIN_D=3 timeout 200 python tools/kv_timing.py >> gpurun_out/t3.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
