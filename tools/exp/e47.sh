cd /root/repo
for p in 0 1 0 1; do PDF_ADAM_L3_LATE=$p timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40; done
