cd /root/repo
NVTX="--nvtx --nvtx-include iters/" bash tools/ncu_box.sh r02w_full_cfg5 'net_adam_x|vl_out|vl_rows|vl_cols|pixel_kernel' 8 -- python tools/prof_step.py --cfg 5 --iters 1
python tools/ncu_sum.py gpurun_out/r02w_full_cfg5.raw.csv > gpurun_out/r02w_full_cfg5_summary.txt
tail -3 gpurun_out/r02w_full_cfg5.log
