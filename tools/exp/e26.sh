cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/timeline.py --cfg 2 2>&1 | grep -E "stages|period" | cut -c1-200
python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40
python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-400
