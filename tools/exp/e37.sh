cd /root/repo
for k in 1 2 4; do echo "ktw=$k $(PDF_GH_KTW=$k timeout 300 python tools/timeline.py --cfg 5 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["period_us"]), d["bwd_l3"][4], d["bwd_l2"][4])')"; done
echo "cfg3 default $(timeout 300 python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-30)"
echo "cfg3 ktw2 $(PDF_GH_KTW=2 timeout 300 python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-30)"
