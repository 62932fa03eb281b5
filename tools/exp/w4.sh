cd /root/repo
for e in "PDF_PRIO=1 PDF_FLIP_MODE=2" "PDF_PRIO=1 PDF_FLIP_MODE=0" "PDF_PRIO=1 PDF_FLIP_MODE=1" "PDF_PRIO=1 PDF_THETA_FLIP=0"; do
echo "== $e"; env $e python tools/timeline.py --cfg 2 2>&1 | grep -v Warn | grep -v nanmean | head -11
done
