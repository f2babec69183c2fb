cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/sgd_check.py > gpurun_out/sgd_check.log 2>&1
timeout 900 python -m pytest tests/test_scale.py tests/test_gpu_parity.py -q -x -m gpu -k "sgd or c4 or scale or solvers or derivative" > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log
timeout 300 python tools/one_step.py C4 1 > gpurun_out/one_step_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file gpurun_out/launches_c4.csv python tools/one_step.py C4 1 > gpurun_out/launches_ncu.log 2>&1
for V in "C1" "C1 simt"; do timeout 300 python tools/cg_parity_variants.py $V >> gpurun_out/cg_variants_c1.log 2>&1; done
