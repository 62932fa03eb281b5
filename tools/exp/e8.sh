cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for d in 3 6; do for wb in 4 8; do
echo "D=$d WB=$wb"
for c in 2 5; do PDF_BWD_D=$d PDF_BWD_WB=$wb python tools/phases.py --cfg $c --iters 5 2>&1 | tail -1 | cut -c60-400; done
done; done
for d in 3 6; do PDF_BWD_D=$d python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-400; done
