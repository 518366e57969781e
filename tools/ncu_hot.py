"""Summarise an ncu report's source page (dev tool): hottest CUDA source lines
by warp-stall samples and executed instructions for one launch.
usage: python tools/ncu_hot.py REPORT.ncu-rep [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = []
fname = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        rows.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"]), fname, r[0],
                     r[1][:90]))
    except (ValueError, KeyError):
        pass
tot = sum(x[0] for x in rows) or 1
toti = sum(x[1] for x in rows) or 1
print(f"total stall samples {tot}, instructions {toti}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {100*i/toti:5.1f}%i {f}:{ln:>4} {src}")
