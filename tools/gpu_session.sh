mkdir -p gpurun_out
timeout 300 python tools/hist_timing.py cfg3 cfg5 > gpurun_out/r2_hist.log 2>&1; echo "hist rc=$?"
cat gpurun_out/r2_hist.log | tail -8
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests.sum --clock-control none --csv --log-file gpurun_out/r2_hist_ncu.csv python tools/hist_timing.py cfg5 > gpurun_out/r2_hist_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_csv.py gpurun_out/r2_hist_ncu.csv 2>/dev/null | tail -10
