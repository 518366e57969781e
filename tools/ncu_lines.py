"""Per-CUDA-line stall breakdown of one launch in an ncu report (dev tool).
usage: python tools/ncu_lines.py REPORT.ncu-rep LAUNCH [file:lo-hi] [min_samples]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
flt = sys.argv[3] if len(sys.argv) > 3 else None
mins = int(sys.argv[4]) if len(sys.argv) > 4 else 5
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
    if r[0] == "Function Name":
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
        cur = {"file": fname, "line": ln, "src": r[1][:80], "samples": 0, "inst": 0, "stalls": {}}
        lines.append(cur)
        continue
    if cur is None:
        continue
    for k, v in zip(hdr, r):
        if k == "Warp Stall Sampling (All Samples)" and v.isdigit():
            cur["samples"] += int(v)
        elif k == "Instructions Executed" and v.isdigit():
            cur["inst"] += int(v)
        elif k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v):
            cur["stalls"][k[6:]] = cur["stalls"].get(k[6:], 0) + int(v)
if flt:
    f, rng = flt.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    lines = [l for l in lines if l["file"] == f and lo <= l["line"] <= hi]
tot = sum(l["samples"] for l in lines)
print(f"samples {tot}")
for l in lines:
    if l["samples"] >= mins:
        top = sorted(l["stalls"].items(), key=lambda kv: -kv[1])[:3]
        print(f"{l['file']}:{l['line']:5d} {l['samples']:6d} {l['inst'] / 148:8.0f}/cta  {l['src'][:60]:60s} {top}")
