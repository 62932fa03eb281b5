"""Aggregate warp-stall samples per CUDA source line from an ncu report
(`ncu -i rep --page source --csv --print-source cuda,sass`).

    python tools/ncu_lines.py REPORT [--launch N] [--top 30]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--launch", type=int, default=0)
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--kernel", default=None, help="regex on the kernel name")
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass",
           "--launch-skip", str(a.launch), "--launch-count", "1"]
    if a.kernel:
        cmd += ["-k", "regex:" + a.kernel]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    f, rows, hdr = None, [], None
    for x in csv.reader(io.StringIO(out)):
        if not x:
            continue
        if x[0] == "File Path":
            f = x[1].split("/")[-1]
        elif x[0] == "Function Name":
            fn = x[1]
        elif x[0] == "Line No":
            hdr = x
        elif x[0] and hdr:
            try:
                rows.append((int(x[4]), f, x[0], x[1].strip()[:90]))
            except ValueError:
                pass
    tot = sum(r[0] for r in rows) or 1
    print(fn, "samples", tot)
    for s, f, l, src in sorted(rows, reverse=True)[: a.top]:
        print(f"{s:7d} {100 * s / tot:5.1f}%  {f}:{l:<5} {src}")


if __name__ == "__main__":
    main()
