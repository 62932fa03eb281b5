cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for x in 0 1; do PDF_FWD_X=$x python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c1-400; done
PDF_FWD_X=1 python tools/phases.py --cfg 3 2>&1 | tail -1 | cut -c1-400
PDF_FWD_X=1 python tools/phases.py --cfg 1 2>&1 | tail -1 | cut -c1-400
