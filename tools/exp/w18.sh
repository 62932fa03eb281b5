cd /root/repo
for e in "PDF_SPLIT_PIXEL=0" "PDF_SPLIT_PIXEL=1"; do
echo "== $e"; env $e python tools/timeline.py --cfg 4 --scenes 256 2>&1 | grep "iteration period\|^pixel \|^view_bwd \|^view_fwd "
env $e python tools/timeline.py --cfg 5 2>&1 | grep "iteration period\|^pixel \|^view_bwd \|^view_fwd "
done
