cd /root/repo
ncu --nvtx --nvtx-include iters/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w7_launches_cfg5.csv -k "regex:view_kernel|pixel_kernel|net_|vl_|data_|gad_" python tools/prof_step.py --cfg 5 --iters 2 > gpurun_out/w7.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(l for l in open('gpurun_out/w7_launches_cfg5.csv') if l.startswith('"')))
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
out=[(r[ki][:50], float(r[vi].replace(',',''))/1000) for r in rows[1:]]
n=len(out)//2
for k,v in out[n:]: print(f"{k:52s} {v:8.1f}")
print("sum", sum(v for _,v in out[n:]))
PY
