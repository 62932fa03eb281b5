cd /root/repo
for e in "PDF_GH_HALF=1" "PDF_GH_HALF=0"; do
echo "== $e"; env $e python tools/timeline.py --cfg 5 2>&1 | grep "^fwd_l\|^bwd_l3\|^bwd_l2\|iteration period" | awk '{print $1, $NF}' | tr '\n' ' '; echo
done
python tools/timeline.py --cfg 3 2>&1 | grep "^fwd_l\|^bwd_l\|iteration period" | awk '{print $1, $NF}' | tr '\n' ' '
