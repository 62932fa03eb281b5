cd /root/repo
bash tools/ncu_box.sh bview "view_kernel|pixel" 3 -- --nvtx --nvtx-include "iters/" --launch-skip 3 python tools/prof_step.py --cfg 4 --scenes 64 --iters 2
python tools/exp/sumraw.py gpurun_out/bview.raw.csv 2>/dev/null | head
