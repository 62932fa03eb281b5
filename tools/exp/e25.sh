cd /root/repo
python tools/timeline.py --cfg 2 2>&1 | grep stages
python tools/timeline.py --cfg 4 --scenes 64 2>&1 | grep -v Warn | tail -14 | head -13
