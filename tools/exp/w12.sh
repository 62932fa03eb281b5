cd /root/repo
NVTX="--nvtx --nvtx-include iters/" bash tools/ncu_box.sh r02w_full_cfg5_net 'net_fwd_mma|net_gh_t' 5 -- python tools/prof_step.py --cfg 5 --iters 1
python tools/ncu_sum.py gpurun_out/r02w_full_cfg5_net.raw.csv > gpurun_out/r02w_full_cfg5_net_summary.txt
