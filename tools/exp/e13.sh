cd /root/repo
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:'net_adam_x|net_gh_x|net_fwd_x|view_kernel|pixel' --launch-skip 300 -c 20 --csv python tools/timeline.py --cfg 2 > gpurun_out/ncu_nc.csv 2> gpurun_out/ncu_nc.err
python tools/launch_summary.py gpurun_out/ncu_nc.csv
grep -E "adam|gh_x" gpurun_out/ncu_nc.csv | head -12 | cut -c1-300
