cd /root/repo
python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_trajectories.py -q -x 2>&1 | tail -2
for s in 4 2; do echo "== cfg5 ADAM_ST=$s"; PDF_ADAM_ST=$s python tools/timeline.py --cfg 5 2>&1 | grep -E "period|^bwd_l1 "; done
for s in 4 2; do echo "== cfg3 ADAM_ST=$s"; PDF_ADAM_ST=$s python tools/timeline.py --cfg 3 2>&1 | grep -E "period|^bwd_l1 "; done
for s in 4 2; do echo "== cfg2 ADAM_ST=$s"; PDF_ADAM_ST=$s python tools/timeline.py --cfg 2 2>&1 | grep -E "period|^bwd_l1 |^fwd_l1 "; done
