cd /root/repo
python -m pytest tests/test_gpu_large.py -x -q 2>&1 | tail -1
python tools/timeline.py --cfg 5 2>&1 | tail -1 | cut -c1-400
python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-120
