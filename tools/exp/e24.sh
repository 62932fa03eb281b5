cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in 2 3; do python tools/timeline.py --cfg $c 2>&1 | tail -1 | cut -c1-40; done
