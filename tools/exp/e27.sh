cd /root/repo
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size --clock-control none --nvtx --nvtx-include "iters/" --csv --log-file gpurun_out/l5.csv python tools/prof_step.py --cfg 5 --iters 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/l5.csv')))
hi=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); h=rows[hi]
ki,mi,vi,idi=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value'),h.index('ID')
per=collections.OrderedDict()
for r in rows[hi+1:]:
    per.setdefault(r[idi],{'k':r[ki]})[r[mi]]=r[vi]
for i,l in per.items():
    print(i, l['k'][:60], l.get('gpu__time_duration.sum'), 'fp64%', l.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'), 'warps%', l.get('sm__warps_active.avg.pct_of_peak_sustained_active'), 'regs', l.get('launch__registers_per_thread'), 'grid', l.get('launch__grid_size'), 'blk', l.get('launch__block_size'))
PY
