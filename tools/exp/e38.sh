cd /root/repo
bash tools/ncu_box.sh bbwd "net_bwd_mma|net_fwd_mma" 2 -- --nvtx --nvtx-include "iters/" --launch-skip 1 python tools/prof_step.py --cfg 4 --scenes 64 --iters 2
