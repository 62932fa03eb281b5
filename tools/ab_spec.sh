cd /root/repo
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in 2 3 1; do for s in 0 1; do echo "== cfg$c SPEC=$s"; PDF_SPEC=$s python tools/timeline.py --cfg $c 2>&1 | grep -E "period|^view_|^pixel "; done; done
