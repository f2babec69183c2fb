#!/usr/bin/env bash
# The one GPU-side runner (run under gpurun; outputs land in gpurun_out/):
#
#   gpurun --timeout 1200 -- 'bash tools/gpu_run.sh tests bench'
#
# Modes (any sequence, executed in order):
#   tests            pytest -m gpu                      -> gpurun_out/pytest_gpu.log
#   smoke            __graft_entry__.smoke()            -> gpurun_out/smoke.log
#   bench            python bench.py $BENCH_ARGS        -> gpurun_out/bench.log
#   reference        python bench.py --impl reference   -> gpurun_out/bench_ref.log
#   launches         ncu launch list of a short bench   -> gpurun_out/launches.csv
#   full             ncu --set full of kernel $KREGEX in `python $SCRIPT`
#                                                       -> gpurun_out/full_$TAG.ncu-rep
#   script           python $SCRIPT                     -> gpurun_out/script_$TAG.log
# Every command runs under its own timeout; ncu runs only after the same
# command exited 0 without it.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-run}
BENCH_ARGS=${BENCH_ARGS:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
for mode in "$@"; do
  case "$mode" in
    tests)
      timeout "${TEST_TIMEOUT:-1500}" python -m pytest tests -m gpu -q -ra -x ${PYTEST_ARGS:-} \
        > gpurun_out/pytest_gpu.log 2>&1
      echo "rc=$?" >> gpurun_out/pytest_gpu.log ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "rc=$?" >> gpurun_out/smoke.log ;;
    bench)
      timeout "${BENCH_TIMEOUT:-1500}" python bench.py $BENCH_ARGS > gpurun_out/bench_$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/bench_$TAG.log ;;
    reference)
      timeout 900 python bench.py --impl reference $BENCH_ARGS > gpurun_out/bench_ref_$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/bench_ref_$TAG.log ;;
    launches)
      LARGS=${LAUNCH_ARGS:---steps 1 --warmup 3 --no-cpu-baseline --no-e2e}
      timeout 900 python bench.py $LARGS > gpurun_out/launches_plain_$TAG.log 2>&1 && \
      timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c ${LAUNCH_COUNT:-20000} --csv \
        --log-file gpurun_out/launches_$TAG.csv python bench.py $LARGS > gpurun_out/launches_ncu_$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/launches_ncu_$TAG.log ;;
    full)
      timeout 900 python $SCRIPT > gpurun_out/full_plain_$TAG.log 2>&1 && \
      timeout 1800 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -s ${SKIP:-1} -c 1 \
        -o gpurun_out/full_$TAG -f python $SCRIPT > gpurun_out/full_ncu_$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/full_ncu_$TAG.log ;;
    script)
      timeout "${SCRIPT_TIMEOUT:-900}" python $SCRIPT > gpurun_out/script_$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/script_$TAG.log ;;
    *) echo "unknown mode $mode" >&2 ;;
  esac
done
