cd /root/repo
for c in 2; do python tools/timeline.py --cfg $c 2>&1 | tail -14 | head -13; done
