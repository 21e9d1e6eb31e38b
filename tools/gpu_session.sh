mkdir -p gpurun_out
timeout 300 python tools/hist_timing.py cfg3 cfg5 > gpurun_out/r2_hist.log 2>&1; echo "hist rc=$?"
cat gpurun_out/r2_hist.log | tail -8
timeout 600 python -m pytest tests/test_gpu_parity.py -k histogram -q -x > gpurun_out/r2_t6.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2_t6.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_hist_ncu3.csv python tools/hist_timing.py cfg3 > /dev/null 2>&1
python tools/ncu_csv.py gpurun_out/r2_hist_ncu3.csv 2>/dev/null | tail -10
