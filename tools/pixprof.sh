# ncu counters of the pixel-mapping kernel on cfg3 / cfg5 (A/B helper)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct
for c in ${CONFIGS:-cfg3 cfg5}; do
python tools/prof_stage.py --config $c --stage map > /dev/null || exit 1
ncu --metrics $M --clock-control none -k regex:pixel_kernel --csv python tools/prof_stage.py --config $c --stage map > gpurun_out/pix_$c.csv 2>&1
done
