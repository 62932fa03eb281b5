# marginal cost of each hot-loop kernel inside the replayed graph (experiment)
for m in 0 1 2 4 8 16 32 128 256 512 1023; do
  out=$(PDF_SKIP_PHASES=$m timeout 120 python tools/phases.py --iters 2 "$@" 2>&1 | tail -1)
  echo "skip=$m $(echo "$out" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["graph_us_per_iter"],1))
except Exception as e: print("ERR", e)')"
done
