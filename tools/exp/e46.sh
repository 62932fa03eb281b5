cd /root/repo
timeout 300 python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-420
timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-40
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
