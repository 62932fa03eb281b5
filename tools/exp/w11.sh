cd /root/repo
NVTX="--nvtx --nvtx-include iters/" bash tools/ncu_box.sh r02w_full_cfg2_pixel 'pixel_kernel' 1 -- python tools/prof_step.py --cfg 2 --iters 1
python tools/ncu_sum.py gpurun_out/r02w_full_cfg2_pixel.raw.csv > gpurun_out/r02w_full_cfg2_pixel_summary.txt
