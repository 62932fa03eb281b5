cd /root/repo
for t in "3 3" "3 6" "3 12" "6 3" "6 6" "12 12"; do set -- $t; echo "tgt=$1 tgt1=$2 $(PDF_BWD_TGT=$1 PDF_BWD_TGT1=$2 python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c60-400)"; done
