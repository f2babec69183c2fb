# ncu --set full (with source) of the refresh operator launch and the
# persistent AP kernel of one C2 AP solve (tools/ap_timing.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/ap_timing.py > gpurun_out/prof_ap_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"kv_tc_kernel|ap_persistent" -c 2 \
  -o gpurun_out/prof_ap_${1:-x} -f python tools/ap_timing.py > gpurun_out/prof_ap_ncu.log 2>&1
tail -3 gpurun_out/prof_ap_ncu.log
