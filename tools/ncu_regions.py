"""Per-region totals of an ncu source page (dev tool): warp-stall samples and
executed instructions per CTA, grouped by the `// ---- phase` markers of
decode.cu. usage: python tools/ncu_regions.py REPORT.ncu-rep [launch_index]"""
import csv
import io
import os
import re
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2411_02886_b200", "csrc",
                   "decode.cu")
marks = []
for i, line in enumerate(open(src), 1):
    m = re.match(r"\s*// ---- (phase \d+[^\n]{0,40})", line)
    if m:
        marks.append((i, m.group(1)))
    m = re.match(r"(__device__|__global__|template).*?\b(\w+)\(", line)
    if m and not line.strip().startswith("//"):
        marks.append((i, "fn " + m.group(2)))
marks.sort()
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
hdr, fname, agg, tot = None, None, {}, [0, 0]
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
        s, n, ln = int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"]), int(r[0])
    except (ValueError, KeyError):
        continue
    key = fname
    if fname == "decode.cu":
        key = "?"
        for mi, name in marks:
            if mi <= ln:
                key = name
    a = agg.setdefault(key, [0, 0])
    a[0] += s
    a[1] += n
    tot[0] += s
    tot[1] += n
print(f"total stall samples {tot[0]}, instructions {tot[1]} ({tot[1] / 148:.0f}/CTA)")
for k, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100 * s / max(tot[0], 1):5.1f}% samples {n / 148:9.0f} instr/CTA  {k}")
