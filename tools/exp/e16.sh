cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/timeline.py --cfg 2 2>&1 | tail -14 | grep -v Warn | grep -v nanmean
python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-30
python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-200
