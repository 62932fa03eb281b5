cd /root/repo
for p in 1 0 1 0; do PDF_ADAM_L2_AFTER=$p timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40; done
timeout 300 python tools/timeline.py --cfg 1 2>&1 | tail -1 | cut -c1-40
timeout 300 python -m pytest tests/test_gpu_trajectories.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
