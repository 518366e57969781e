"""Stall-reason totals and the top source lines of one launch in an ncu report
(dev tool). usage: python tools/ncu_stalls.py REPORT LAUNCH [n_top]"""
import collections
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
fname, hdr, cur = None, None, None
lines = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] != "":
        try:
            ln = int(r[0])
        except ValueError:
            continue
        cur = {"file": fname, "line": ln, "src": r[1][:70], "samples": 0, "stalls": collections.Counter()}
        lines.append(cur)
        continue
    if cur is None:
        continue
    for k, v in zip(hdr, r):
        if k == "Warp Stall Sampling (All Samples)" and v.isdigit():
            cur["samples"] += int(v)
        elif k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v):
            cur["stalls"][k[6:]] += int(v)
tot = collections.Counter()
for l in lines:
    tot.update(l["stalls"])
print("samples", sum(l["samples"] for l in lines), "stall totals:", tot.most_common(14))
for l in sorted(lines, key=lambda l: -l["samples"])[:ntop]:
    print(f"{l['file']}:{l['line']:5d} {l['samples']:6d}  {l['src']:70s} {l['stalls'].most_common(3)}")
