cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_trajectories.py tests/test_gpu_sharded.py -m gpu -q -x 2>&1 | tail -5
python tools/timeline.py --cfg 2 2>&1 | grep -v Warn | grep -v nanmean | grep "iteration period\|^pixel"
python tools/timeline.py --cfg 3 2>&1 | grep -v Warn | grep -v nanmean | grep "iteration period\|^pixel"
python tools/timeline.py --cfg 1 2>&1 | grep -v Warn | grep -v nanmean | grep "iteration period\|^pixel"
