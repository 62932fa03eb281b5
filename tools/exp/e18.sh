cd /root/repo
python -m pytest tests/test_gpu_large.py tests/test_gpu_trajectories.py -x -q 2>&1 | tail -1
for c in 2 3 5; do python tools/timeline.py --cfg $c 2>&1 | tail -1 | cut -c1-700; done
