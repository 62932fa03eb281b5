cd /root/repo
for g in 10 50 10 50; do PDF_GRAPH_ITERS=$g timeout 600 python bench.py --steps 3 --warmup 3 --batch 0 --large-iters 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($g, round(d['value']), round(d['e2e']['value']))"; done
