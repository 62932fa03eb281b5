#!/bin/bash
# One GPU-box profiling session (run through gpurun): bench line, ncu launch lists of the
# cfg2 / cfg4 / cfg5 training loops, and full-set captures of the dominant training kernels
# (NVTX range "iters" of tools/prof_step.py: the fixture synthesis and init are excluded).
#   bash tools/prof_round.sh TAG [bench|lists|full|all]
tag=${1:-r02}; what=${2:-all}
cd /root/repo; mkdir -p gpurun_out
out=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
K="regex:view_kernel|pixel_kernel|pix_|net_|vl_|data_|gad_"
NV="--nvtx --nvtx-include iters/"
if [[ $what == bench || $what == all ]]; then
  python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc=$?"
fi
if [[ $what == lists || $what == all ]]; then
  for c in "2 1" "4 256" "5 1"; do set -- $c
    ncu $NV --metrics $M --clock-control none --csv --log-file $out/${tag}_launches_cfg$1.csv -k "$K" \
      python tools/prof_step.py --cfg $1 --scenes $2 --iters 10 --graph > $out/${tag}_ncu_cfg$1.log 2>&1
    echo "ncu cfg$1 rc=$?"; gzip -f $out/${tag}_launches_cfg$1.csv
  done
fi
if [[ $what == full || $what == all ]]; then
  NVTX="$NV" bash tools/ncu_box.sh ${tag}_full_cfg4 'pix_|pixel_kernel|view_kernel|net_bwd_mma|net_fwd_mma' 11 -- \
    python tools/prof_step.py --cfg 4 --scenes 256 --iters 1 ; echo "full cfg4 rc=$?"
  NVTX="$NV" bash tools/ncu_box.sh ${tag}_full_cfg5 'vl_|net_adam_x|net_gh_|net_fwd|pix_|pixel_kernel|data_' 24 -- \
    python tools/prof_step.py --cfg 5 --iters 1 ; echo "full cfg5 rc=$?"
  NVTX="$NV" bash tools/ncu_box.sh ${tag}_full_cfg2 'view_kernel|pixel_kernel|net_|data_|gad_' 12 -- \
    python tools/prof_step.py --cfg 2 --iters 1 ; echo "full cfg2 rc=$?"
fi
ls -la $out | tail -40
