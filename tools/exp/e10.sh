cd /root/repo
run() { echo "$1: $(env $1 python tools/timeline.py --cfg 2 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["period_us"],1), {k: v[4] for k, v in d.items() if k.startswith("bwd")})')"; }
run "PDF_BWD_CLUSTER=16"
run "PDF_BWD_CLUSTER=8"
run "PDF_BWD_CLUSTER=4"
run "PDF_BWD_CLUSTER=2"
run "PDF_BWD_KT=2"
run "PDF_BWD_KT=2 PDF_BWD_CLUSTER=8"
run "PDF_BWD_TGT=6 PDF_BWD_TGT1=6"
run "PDF_BWD_WB=4"
