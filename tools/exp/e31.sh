cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/e2e_breakdown.py --cfg 2 2>&1 | tail -12
