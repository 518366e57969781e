"""Static SASS instructions of the fused decode kernel per source region
(dev tool: the post-scan phases run once per launch from a cold instruction
cache, so their code size is latency). usage: python tools/code_size.py [D G [LEAN]]"""
import bisect
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D, G = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("128", "4")
LEAN = sys.argv[3] if len(sys.argv) > 3 else "1"
obj = os.path.join(ROOT, "paper_2411_02886_b200", "_build", "decode.cu.o")
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=td, capture_output=True)
    cubin = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(td, cubin)], capture_output=True, text=True).stdout
name = f"decode_kernelILi{D}ELi{G}ELb1ELb{LEAN}EEEvNS_12DecodeParamsE:"
start = dis.index(name)
body = dis[start:]
end = body.find("//---------------------", 10)
body = body[: end if end > 0 else None]
line_re = re.compile(r'//## File "([^"]+)", line (\d+)')
addr_re = re.compile(r"/\*([0-9a-f]{4,})\*/")
counts, key = {}, None
for l in body.split("\n"):
    m = line_re.search(l)
    if m:
        key = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if key and addr_re.search(l):
        counts[key] = counts.get(key, 0) + 1
src = open(os.path.join(ROOT, "paper_2411_02886_b200", "csrc", "decode.cu")).read().split("\n")
marks = [(i, l.strip()[:70]) for i, l in enumerate(src, 1)
         if re.match(r"\s*// ---- phase", l) or re.match(r"(__device__|__global__)", l)]
agg = {}
for (f, ln), c in counts.items():
    if f != "decode.cu":
        k = f
    else:
        i = bisect.bisect_right([m[0] for m in marks], ln) - 1
        k = marks[i][1] if i >= 0 else "?"
    agg[k] = agg.get(k, 0) + c
print("total instructions", sum(agg.values()))
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:25]:
    print(f"{v:6d}  {k}")
