"""Summarise ncu outputs into a committed text file under profiles/ (dev tool).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv      # launch list -> per-kernel shares
    python tools/summarize_ncu.py full gpurun_out/prof_decode.ncu-rep    # --set full -> key counters per launch
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = OrderedDict()
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        agg.setdefault(name, []).append(float(d["Metric Value"]))
    unit = "ns"
    tot = sum(sum(v) for v in agg.values())
    print(f"# launch list ({path}); times in {unit}, cold-cache serialised (compare shares)")
    print(f"{'launches':>8} {'mean':>12} {'total':>14} {'share':>7}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v):12.1f} {sum(v):14.1f} {100 * sum(v) / tot:6.1f}%  {k}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full ({path})")
    for n, r in enumerate(rows[2:]):
        print(f"## launch {n}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:62s} {r[i]} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
