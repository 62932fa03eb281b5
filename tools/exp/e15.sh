cd /root/repo
for cs in 8 16; do PDF_VIEW_CLUSTER=$cs python tools/timeline.py --cfg 2 2>&1 | tail -14 | grep -v Warn | grep -v nanmean; done
PDF_VIEW_CLUSTER=16 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
