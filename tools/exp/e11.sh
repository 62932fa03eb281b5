cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/timeline.py --cfg 2 2>&1 | tail -11
python tools/timeline.py --cfg 5 2>&1 | tail -1
