cd /root/repo
for env in "" "PDF_DATA_GEMM=1"; do echo "cfg4 $env"; env $env python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-330; done
