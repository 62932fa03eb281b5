cd /root/repo
python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_trajectories.py -q -x 2>&1 | tail -2
for p in 0 1; do echo "== cfg5 ADAM_PERSIST=$p"; PDF_ADAM_PERSIST=$p python tools/timeline.py --cfg 5 2>&1 | grep -E "period|^bwd_l1 "; done
echo "== cfg2"; python tools/timeline.py --cfg 2 2>&1 | grep -E "period|^view_|stages"
echo "== cfg3"; for p in 0 1; do PDF_ADAM_PERSIST=$p python tools/timeline.py --cfg 3 2>&1 | grep -E "period|^bwd_l1 "; done
