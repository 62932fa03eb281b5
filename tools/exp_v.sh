cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in 2 3; do echo "cfg$c"; python tools/phases.py --cfg $c 2>&1 | tail -1 | cut -c60-300; done
echo cfg2-nodg; PDF_DATA_GEMM=0 python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c60-300
echo cfg4; python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-300
echo cfg5; python tools/phases.py --cfg 5 --iters 5 2>&1 | tail -1 | cut -c60-300
