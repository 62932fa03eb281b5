cd /root/repo
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in 2 3; do timeout 300 python tools/timeline.py --cfg $c 2>&1 | tail -1 | cut -c1-40; done
timeout 300 python tools/timeline.py --cfg 2 2>&1 | grep "view_bwd " | head -2
timeout 300 python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-300
