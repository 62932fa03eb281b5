cd /root/repo
for m in 36 48 72 96 144; do echo "== PDF_SPEC_MIB=$m"; PDF_SPEC_MIB=$m python tools/timeline.py --cfg 5 2>&1 | grep "iteration period\|^view" | awk '{print $1,$2,$3,$NF}' | tr '\n' ' '; echo; done
