cd /root/repo
for mib in 48 32 72 96; do echo "spec=$mib $(PDF_SPEC_MIB=$mib timeout 300 python tools/timeline.py --cfg 5 2>&1 | tail -1 | cut -c1-30)"; done
