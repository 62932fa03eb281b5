cd /root/repo
echo cfg5; python tools/phases.py --cfg 5 --iters 5 2>&1 | tail -1 | cut -c60-300
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
