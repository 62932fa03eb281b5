cd /root/repo
for e in "PDF_PIX_CHUNK_MIB=40" "PDF_PIX_CHUNK_MIB=20" "PDF_PIX_CHUNK_MIB=80" "PDF_PIX_CHUNK_MIB=100000"; do
echo "== $e"; env $e python tools/timeline.py --cfg 4 --scenes 256 2>&1 | grep "iteration period\|^pixel "
done
