cd /root/repo
for e in "PDF_DATA_FORK=0" "PDF_ADAM_FORK=0" "PDF_PDL=0"; do
echo "== $e"; env $e python tools/timeline.py --cfg 2 2>&1 | grep -v Warn | grep -v nanmean | grep "iteration period\|^view\|^pixel"
done
