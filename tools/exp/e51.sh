cd /root/repo
bash tools/ncu_box.sh adam5 "net_adam_x|net_gh_t" 3 -- --nvtx --nvtx-include "iters/" python tools/prof_step.py --cfg 5 --iters 2
