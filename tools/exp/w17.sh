cd /root/repo
NVTX="--nvtx --nvtx-include iters/" bash tools/ncu_box.sh r02w_solo 'view_kernel' 2 -- python tools/prof_step.py --cfg 4 --scenes 256 --iters 1
python tools/ncu_sum.py gpurun_out/r02w_solo.raw.csv > gpurun_out/r02w_solo_summary.txt
