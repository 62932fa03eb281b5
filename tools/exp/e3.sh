cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash tools/skip_sweep.sh --cfg 2
