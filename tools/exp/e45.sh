cd /root/repo
bash tools/ncu_box.sh bbwd2 "net_bwd_mma" 3 -- --nvtx --nvtx-include "iters/" python tools/prof_step.py --cfg 4 --scenes 64 --iters 2
