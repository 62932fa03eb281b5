cd /root/repo
run() { echo "$1: $(env $1 timeout 300 python tools/phases.py --cfg 4 --scenes 128 --iters 3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); p=d["phases_us"]; print(round(d["graph_us_per_iter"]), p["view_fwd"], p["pixel"], p["view_bwd"])')"; }
run "PDF_X=0"
run "PDF_DATA_GEMM=0"
run "PDF_VIEW_CLUSTER=8"
run "PDF_PIX_WARPS=4"
run "PDF_BWD_CLUSTER=8"
