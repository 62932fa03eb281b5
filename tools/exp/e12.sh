cd /root/repo
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 1 2; do python tools/timeline.py --cfg $c 2>&1 | tail -11 | head -10; done
