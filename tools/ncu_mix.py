"""Instruction mix and headline metrics of one ncu capture (a .ncu-rep file).

    python tools/ncu_mix.py gpurun_out/prof.ncu-rep [--top 24]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 24
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
keys = ("Duration", "Executed Instructions", "Issue Slots Busy", "Registers Per Thread", "Achieved Active Warps",
        "Warp Cycles Per Issued", "Eligible Warps Per", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Memory Throughput")
for line in det.splitlines():
    if any(k in line for k in keys):
        print(line.strip())
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ie, sc = hdr.index("Instructions Executed"), hdr.index("Source")
tot, ops = 0, collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    tot += n
    t = r[sc].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    ops[op.split(".")[0]] += n
print(f"warp instructions executed: {tot / 1e6:.1f} M")
for k, v in ops.most_common(top):
    print(f"  {k:10s} {v / 1e6:8.2f} M {100 * v / tot:5.1f} %")
