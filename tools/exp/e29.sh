cd /root/repo
run() { echo "$1: $(env $1 python tools/phases.py --cfg 4 --scenes 128 --iters 5 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); p=d["phases_us"]; print(round(d["graph_us_per_iter"]), {k: p[k] for k in ("fwd_l2","bwd_l3","bwd_l2","bwd_l1")})')"; }
run "PDF_X=0"
run "PDF_BWD_KT=1"
run "PDF_BWD_KT=1 PDF_BWD_D=6"
run "PDF_BWD_KT=1 PDF_BWD_WB=4 PDF_BWD_D=6"
run "PDF_BWD_WB=4"
run "PDF_FWD_NT=2"
run "PDF_BWD_TGT=6"
