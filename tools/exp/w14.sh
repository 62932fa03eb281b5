cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -m gpu -q -x 2>&1 | tail -2
python tools/timeline.py --cfg 2 2>&1 | grep "iteration period\|^view"
python tools/timeline.py --cfg 4 --scenes 256 2>&1 | grep "iteration period\|^view\|^pixel"
python tools/timeline.py --cfg 3 2>&1 | grep "iteration period\|^view"
