cd /root/repo
for i in 1 2; do python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40; done
PDF_ADAM_FORK=0 python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40
PDF_BWD_X=0 python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40
python tools/timeline.py --cfg 3 2>&1 | tail -13 | head -10
