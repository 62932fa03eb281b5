cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 2 3 5; do python tools/timeline.py --cfg $c 2>&1 | tail -1 | cut -c1-40; done
