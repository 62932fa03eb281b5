"""Per-kernel summary of an ncu launch list (`ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X`), gzipped or not.

    python tools/launch_summary.py profiles/r01g_launches_cfg2.csv.gz
"""
import collections
import csv
import gzip
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, idi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        per[r[idi]]["k"] = r[ki]
        per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for launch in per.values():
        a = agg[launch["k"].split("(")[0].replace("void ", "")]
        a[0] += 1
        a[1] += launch.get("gpu__time_duration.sum", 0.0)
        a[2] += launch.get("dram__bytes_read.sum", 0.0) + launch.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"launches {len(per)}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{a[0]:5d} {a[1]:10.1f} us {100 * a[1] / tot:5.1f}%  avg {a[1] / a[0]:7.2f} us  "
              f"dram/launch {a[2] / a[0] / 1e6:8.2f} MB  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
