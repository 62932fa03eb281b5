cd /root/repo
for w in 8 4; do echo "w=$w $(PDF_PIX_WARPS=$w timeout 300 python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["graph_us_per_iter"]), d["phases_us"]["pixel"])')"; done
for w in 8 4; do echo "cfg5 w=$w $(PDF_PIX_WARPS=$w timeout 300 python tools/phases.py --cfg 5 --iters 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["graph_us_per_iter"]), d["phases_us"]["pixel"])')"; done
PDF_PIX_WARPS=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
