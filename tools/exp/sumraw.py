import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[0]; units=rows[1]
want=['Kernel Name','gpu__time_duration.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum','dram__bytes_write.sum','launch__grid_size','launch__block_size','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed','sm__cycles_active.avg']
idx=[hdr.index(w) if w in hdr else None for w in want]
for r in rows[2:]:
    print(' | '.join((r[i][:40] if i is not None else '-') + ('' if i is None else units[i]) for i in idx))
