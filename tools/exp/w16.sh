cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_trajectories.py tests/test_gpu_edges.py -m gpu -q -x 2>&1 | tail -3
PDF_VIEW_CLUSTER=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -m gpu -q -x 2>&1 | tail -3
python tools/timeline.py --cfg 4 --scenes 256 2>&1 | grep "iteration period\|^view\|^pixel"
PDF_VIEW_CLUSTER=4 python tools/timeline.py --cfg 4 --scenes 256 2>&1 | grep "iteration period\|^view\|^pixel"
