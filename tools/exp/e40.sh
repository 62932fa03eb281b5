cd /root/repo
bash tools/ncu_box.sh full2 "net_|view_kernel|pixel" 9 -- --nvtx --nvtx-include "iters/" --launch-skip 9 python tools/prof_step.py --cfg 2 --iters 3
python tools/ncu_sum.py gpurun_out/full2.raw.csv > gpurun_out/full2.sum.txt 2>&1
