cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/sgd_check.py > gpurun_out/sgd_check.log 2>&1; echo "rc=$?" >> gpurun_out/sgd_check.log
if grep -q "C4 epoch" gpurun_out/sgd_check.log; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_slab -s 20 -c 1 -o gpurun_out/full_sgd_lazy2 -f python tools/sgd_timing.py 393216 1 > gpurun_out/ncu_lazy2.log 2>&1
fi
for V in "C3" "C3 simt" "C1" "C1 simt"; do
  for E in "" "GPK_TGRAM=0" "GPK_FLUSH_CHUNKS=4" "GPK_DENSE_CAP=0"; do
    case "$V$E" in C3*GPK_DENSE_CAP*) continue;; esac
    env $E timeout 300 python tools/cg_parity_variants.py $V >> gpurun_out/cg_variants.log 2>&1
  done
done
timeout 1200 python tools/make_golden_scale.py validate > gpurun_out/golden_validate.log 2>&1; echo "rc=$?" >> gpurun_out/golden_validate.log
