cd /root/repo
for env in "PDF_DATA_GEMM=0" "PDF_DATA_GEMM=0 PDF_EXP_NODATA=1" "PDF_DATA_GEMM=1"; do echo "$env"; env $env python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c60-250; done
