cd /root/repo
python tools/timeline.py --cfg 2 2>&1 | tail -12
python tools/timeline.py --cfg 5 2>&1 | tail -12
