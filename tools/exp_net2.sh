cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for env in "" "PDF_BWD_CLUSTER=8" "PDF_BWD_KT=2"; do
for c in 2 3; do echo "cfg$c $env"; env $env python tools/phases.py --cfg $c 2>&1 | tail -1 | cut -c60-400; done
done
for env in "" "PDF_BWD_KT=1"; do echo "cfg4 $env"; env $env python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-400; done
python tools/phases.py --cfg 5 --iters 5 2>&1 | tail -1 | cut -c60-400
