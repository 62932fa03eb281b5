cd /root/repo
echo "cfg4"; python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-330
echo "cfg2"; python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c60-330
echo "cfg3"; python tools/phases.py --cfg 3 2>&1 | tail -1 | cut -c60-330
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
