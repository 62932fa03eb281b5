cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for nt in 4 2 1; do echo "NT=$nt"; PDF_FWD_NT=$nt python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c90-200; done
echo cfg2; python tools/phases.py --cfg 2 2>&1 | tail -1 | cut -c60-200
echo cfg3; python tools/phases.py --cfg 3 2>&1 | tail -1 | cut -c60-200
echo cfg5; python tools/phases.py --cfg 5 --iters 3 2>&1 | tail -1 | cut -c60-200
