cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "inverse or ap or golden" 2>&1 | tail -1; GPK_PHASE_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep set_hyper | tail -1; timeout 300 python bench.py --no-cpu-baseline 2>&1 | cut -c1-200; } > gpurun_out/quick.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r18.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/quick.log
