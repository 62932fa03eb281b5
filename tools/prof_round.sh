#!/bin/bash
# One GPU-box profiling session (run through gpurun): bench line, ncu launch lists of the
# cfg2 / cfg4 / cfg5 legs, and full-set captures of the dominant kernels.
#   bash tools/prof_round.sh TAG
tag=${1:-r02}
cd /root/repo
out=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
K="regex:view_kernel|pixel_kernel|net_|vl_|data_|gad_"
python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc=$?"
ncu --metrics $M --clock-control none --csv --log-file $out/${tag}_launches_cfg2.csv -k "$K" \
  python bench.py --steps 1 --warmup 3 --iters 20 --batch 0 --large-iters 0 --no-cpu-baseline --no-timeline \
  > $out/${tag}_ncu_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"
ncu --metrics $M --clock-control none --csv --log-file $out/${tag}_launches_cfg4.csv -k "$K" \
  python tools/prof_step.py --cfg 4 --scenes 256 --iters 10 --graph > $out/${tag}_ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
ncu --metrics $M --clock-control none --csv --log-file $out/${tag}_launches_cfg5.csv -k "$K" \
  python tools/prof_step.py --cfg 5 --iters 10 --graph > $out/${tag}_ncu_cfg5.log 2>&1; echo "ncu cfg5 rc=$?"
for f in $out/${tag}_launches_*.csv; do gzip -f $f; done
bash tools/ncu_box.sh ${tag}_full_cfg4 'pixel_kernel|view_kernel|net_bwd_mma|net_fwd_mma' 6 -- \
  python tools/prof_step.py --cfg 4 --scenes 256 --iters 1 ; echo "full cfg4 rc=$?"
bash tools/ncu_box.sh ${tag}_full_cfg5 'vl_|net_adam_x|net_gh_x|pixel_kernel' 8 -- \
  python tools/prof_step.py --cfg 5 --iters 1 ; echo "full cfg5 rc=$?"
bash tools/ncu_box.sh ${tag}_full_cfg2 'view_kernel|pixel_kernel|net_' 10 -- \
  python tools/prof_step.py --cfg 2 --iters 1 ; echo "full cfg2 rc=$?"
ls -la $out | tail -40
