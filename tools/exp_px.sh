cd /root/repo
echo cfg2; python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c60-300
echo cfg4; python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-300
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
