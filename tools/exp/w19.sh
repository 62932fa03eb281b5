cd /root/repo
python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_edges.py tests/test_gpu_trajectories.py -m gpu -q -x 2>&1 | tail -5
for e in "PDF_PIX_STREAM=1" "PDF_PIX_STREAM=0"; do
echo "== $e"; env $e python tools/timeline.py --cfg 4 --scenes 256 2>&1 | grep "iteration period\|^pixel \|^view_bwd "
env $e python tools/timeline.py --cfg 5 2>&1 | grep "iteration period\|^pixel \|^view_bwd "
done
