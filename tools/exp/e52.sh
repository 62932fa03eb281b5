cd /root/repo
timeout 300 python tools/timeline.py --cfg 5 2>&1 | tail -1 | cut -c1-40
timeout 300 python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40
