cd /root/repo
timeout 300 python -m pytest tests/test_gpu_large.py tests/test_gpu_trajectories.py -x -q 2>&1 | tail -1
timeout 300 python tools/timeline.py --cfg 5 2>&1 | tail -1 | cut -c1-500
timeout 300 python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40
