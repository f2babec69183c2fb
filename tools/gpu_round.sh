#!/usr/bin/env bash
# Round evidence in one gpurun call (outputs in gpurun_out/):
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh'
# 1. pytest -m gpu   2. smoke()   3. default bench.py (C4, N=1)
# 4. ncu launch list of one C4 step (tools/one_step.py)  5. ncu --set full of the SGD slab kernel
# 6. ncu --set full of the SGD finish kernel and the C4 gradient pass
# Each ncu pass runs only after the same command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r02}
[ -n "${SKIP_TESTS:-}" ] || bash tools/gpu_run.sh tests smoke
TAG=$TAG bash tools/gpu_run.sh bench
timeout 600 python tools/one_step.py C4 1 > gpurun_out/one_step_plain_$TAG.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file gpurun_out/launches_C4_$TAG.csv python tools/one_step.py C4 1 > gpurun_out/launches_ncu_$TAG.log 2>&1
timeout 300 python tools/sgd_timing.py 393216 1 > gpurun_out/sgd_timing_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_slab64_kernel -s 20 -c 1 \
  -o gpurun_out/full_sgd_slab_$TAG -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_slab_$TAG.log 2>&1

# 6. ncu --set full of the SGD finish kernel and of the gradient pass of one C4 step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_finish_kernel -s 20 -c 1 \
  -o gpurun_out/full_sgd_finish_$TAG -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_finish_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grad_tc_kernel -c 1 \
  -o gpurun_out/full_grad_tc_$TAG -f python tools/one_step.py C4 1 > gpurun_out/ncu_grad_$TAG.log 2>&1

echo done
