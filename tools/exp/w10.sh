cd /root/repo
for xp in 0 1 17 2 4 8 15; do
echo "== PDF_XP=$xp"; PDF_XP=$xp python tools/timeline.py --cfg 2 2>&1 | grep "^view_fwd\|^view_bwd\|iteration period"
done
