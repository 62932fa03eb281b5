cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 1 2 3; do python tools/phases.py --cfg $c 2>&1 | tail -1 | cut -c60-400; done
python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-400
