"""Summarise one round of GPU captures into profiles/: the bench line (with the ncu DRAM
traffic), the per-launch list and the fused kernel's ncu metrics / source lines.

    python tools/profiles_refresh.py <tag>   # reads gpurun_out/{bench,launches,prof_fused}_<tag>.*
"""

import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    tag = sys.argv[1]
    rep = os.path.join(OUT, f"prof_fused_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
            "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    vals = {w: (u[h.index(w)], v[h.index(w)]) for w in want if w in h}
    with open(os.path.join(PROF, f"r01_k_eval_fused_{tag}_raw.txt"), "w") as f:
        f.write("".join(f"{w} {a} {b}\n" for w, (a, b) in vals.items()))
    rd = float(vals["dram__bytes_read.sum"][1]) * UNIT[vals["dram__bytes_read.sum"][0]]
    wr = float(vals["dram__bytes_write.sum"][1]) * UNIT[vals["dram__bytes_write.sum"][0]]
    tpath = os.path.join(PROF, "ncu_traffic.json")
    t = json.load(open(tpath))
    t["c3"] = {"kernel": "k_eval_fused", "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
               "source": f"profiles/r01_k_eval_fused_{tag}_raw.txt"}
    json.dump(t, open(tpath, "w"), indent=2)
    details = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(os.path.join(PROF, f"r01_k_eval_fused_{tag}_details.txt"), "w").write(details)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    tmp = os.path.join(OUT, f"src_{tag}.csv")
    open(tmp, "w").write(src)
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "30"],
                           capture_output=True, text=True).stdout
    open(os.path.join(PROF, f"r01_k_eval_fused_{tag}_lines.txt"), "w").write(lines)
    # bench line
    line = open(os.path.join(OUT, f"bench_{tag}.json")).read().strip().splitlines()[-1]
    d = json.loads(line)
    d["roofline"]["traffic"] = int(rd + wr)
    open(os.path.join(PROF, "r01_bench_line.json"), "w").write(json.dumps(d) + "\n")
    # launch list
    tot, cnt = collections.defaultdict(float), collections.Counter()
    hdr = None
    for x in csv.reader(open(os.path.join(OUT, f"launches_{tag}.csv"))):
        if not x:
            continue
        if x[0] == "ID":
            hdr = x
            continue
        if hdr is None:
            continue
        dd = dict(zip(hdr, x))
        if dd.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", dd["Kernel Name"])
        val = float(dd["Metric Value"].replace(",", ""))
        un = dd["Metric Unit"]
        val = val / 1000 if un in ("nsecond", "ns") else (val * 1000 if un == "msecond" else val)
        tot[name] += val
        cnt[name] += 1
    T = sum(tot.values())
    fk = [k for k in tot if "k_eval_fused" in k][0]
    pk = [k for k in tot if "k_post" in k][0]
    with open(os.path.join(PROF, f"r01_launches_{tag}.txt"), "w") as f:
        f.write("launch list of `python bench.py --steps 2 --warmup 3 --no-register --cpu-budget 0` "
                "(256^3/64^3, f32)\nncu --metrics gpu__time_duration.sum --clock-control none "
                "(cold-cache, serialised per launch)\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            f.write(f"{k[:66]:66s} launches {cnt[k]:3d} total {tot[k]:9.1f} us  per launch "
                    f"{tot[k] / cnt[k]:8.1f} us  share {tot[k] / T * 100:5.1f}%\n")
        f.write("k_ref_terms / k_pack_rt run once per level (setup), the rest once per evaluation:\n")
        f.write(f"fused share of one evaluation = {tot[fk] / (tot[fk] + tot[pk]) * 100:.1f}%\n")
    print(json.dumps({k: d[k] for k in ("value", "ms_per_step", "e2e")}), d["roofline"]["kernel_ms"],
          d["roofline"]["frac"], d["full_registration"]["seconds"])
    print(open(os.path.join(PROF, f"r01_launches_{tag}.txt")).read())
    print("".join(f"{w} {a} {b}\n" for w, (a, b) in vals.items()))


if __name__ == "__main__":
    main()
