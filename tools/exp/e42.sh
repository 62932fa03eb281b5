cd /root/repo
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for p in 1 0; do PDF_L2_PERSIST=$p timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40; done
for p in 1 0; do PDF_L2_PERSIST=$p timeout 300 python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40; done
for p in 1 0; do PDF_L2_PERSIST=$p timeout 300 python tools/timeline.py --cfg 5 2>&1 | tail -1 | cut -c1-40; done
