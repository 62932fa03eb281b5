cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3; do python tools/timeline.py --cfg $c 2>&1 | tail -1 | cut -c1-40; done
PDF_ADAM_FORK=0 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40
python tools/timeline.py --cfg 2 2>&1 | tail -13 | head -10
