cd /root/repo
timeout 300 python -m pytest tests/test_gpu_large.py -x -q -k "side_branches or split" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for p in 1 0; do PDF_DEFER_ADAM1=$p timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40; done
for p in 1 0; do PDF_DEFER_ADAM1=$p timeout 300 python tools/timeline.py --cfg 1 2>&1 | tail -1 | cut -c1-40; done
