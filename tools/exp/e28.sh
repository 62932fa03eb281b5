cd /root/repo
for bx in 1 2; do PDF_BWD_X=$bx python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | cut -c60-420; done
