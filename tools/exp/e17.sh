cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 1 2 3 5; do python tools/timeline.py --cfg $c 2>&1 | tail -1 | cut -c1-700; done
