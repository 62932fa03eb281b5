cd /root/repo
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for mc in 4 1; do PDF_FWD_MC=$mc timeout 300 python tools/timeline.py --cfg 2 2>&1 | tail -1 | cut -c1-300; done
