cd /root/repo
timeout 300 python -m pytest tests/test_gpu_large.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/timeline.py --cfg 5 2>&1 | tail -1 | cut -c1-30; done
PDF_SPEC_MIB=48 timeout 300 python tools/timeline.py --cfg 5 2>&1 | tail -1 | cut -c1-30
