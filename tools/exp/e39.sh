cd /root/repo
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 2 --warmup 3 --large-iters 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['batched']['scenes_per_s'], d['batched']['e2e_scenes_per_s'])"
