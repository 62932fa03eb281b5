cd /root/repo
NVTX="--nvtx --nvtx-include iters/" bash tools/ncu_box.sh r02w_full_cfg4 'net_bwd_mma|pixel_kernel|view_kernel' 6 -- python tools/prof_step.py --cfg 4 --scenes 256 --iters 1
python tools/ncu_sum.py gpurun_out/r02w_full_cfg4.raw.csv > gpurun_out/r02w_full_cfg4_summary.txt
tail -2 gpurun_out/r02w_full_cfg4.log
