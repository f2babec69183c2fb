cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/ap_timing.py > gpurun_out/ap_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ap_persistent -s 1 -c 1 -o gpurun_out/ap_full -f \
    python tools/ap_timing.py > gpurun_out/ncu_ap.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_ap.log
