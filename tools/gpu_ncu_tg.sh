cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/kv_timing.py 16384 26 65 > gpurun_out/kvt.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_tc_kernel -s 2 -c 1 -o gpurun_out/kv_tg -f \
    python tools/kv_timing.py 16384 26 65 > gpurun_out/ncu_kvtg.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_kvtg.log
GPK_TGRAM=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_tc_kernel -s 2 -c 1 -o gpurun_out/kv_notg -f \
    python tools/kv_timing.py 16384 26 65 >> gpurun_out/ncu_kvtg.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_kvtg.log
