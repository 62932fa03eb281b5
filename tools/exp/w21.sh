cd /root/repo
NVTX="--nvtx --nvtx-include iters/" bash tools/ncu_box.sh r02y_pix 'pix_' 3 -- python tools/prof_step.py --cfg 4 --scenes 256 --iters 1
python tools/ncu_sum.py gpurun_out/r02y_pix.raw.csv > gpurun_out/r02y_pix_summary.txt
NVTX="--nvtx --nvtx-include iters/" bash tools/ncu_box.sh r02y_pix5 'pix_' 3 -- python tools/prof_step.py --cfg 5 --iters 1
python tools/ncu_sum.py gpurun_out/r02y_pix5.raw.csv > gpurun_out/r02y_pix5_summary.txt
