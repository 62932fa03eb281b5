cd /root/repo
python -m pytest tests/test_gpu_large.py tests/test_gpu_properties.py -m gpu -q -x 2>&1 | tail -3
python tools/timeline.py --cfg 5 2>&1 | grep "iteration period\|^view"
