cd /root/repo
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'view_kernel|pixel_kernel|net_|set_ints|vl_|data_' --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --steps 1 --warmup 3 --iters 20 --batch 0 --large-iters 0 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu=$?
gzip -f gpurun_out/launches_cfg2.csv
