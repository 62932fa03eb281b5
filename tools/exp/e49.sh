cd /root/repo
for mc in 2 4 2 4; do PDF_FWD_MC=$mc timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40; done
PDF_FWD_MC=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
