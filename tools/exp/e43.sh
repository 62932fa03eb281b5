cd /root/repo
for p in 1 0; do PDF_STREAM_PRIO=$p timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40; done
for p in 1 0; do PDF_STREAM_PRIO=$p timeout 300 python tools/timeline.py --cfg 1 2>&1 | tail -1 | cut -c1-40; done
timeout 300 python tools/timeline.py --cfg 2 2>&1 | grep -v Warn | grep -v nanmean | tail -14 | head -10
