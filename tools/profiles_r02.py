"""Summarise the round-2 captures into profiles/: the launch list of the bench's
evaluation loop, the lean march's ncu metrics, details, instruction mix and source lines,
the post kernel's details, and the DRAM traffic the bench reports as roofline.traffic.

    python tools/profiles_r02.py   # reads gpurun_out/{launches_final.csv,prof_final,prof_post_final}
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


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep = os.path.join(OUT, "prof_final.ncu-rep")
    r = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    h, u, v = r[0], r[1], r[2]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
            "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__throughput.avg.pct_of_peak_sustained_active"]
    vals = {w: (u[h.index(w)], v[h.index(w)]) for w in want if w in h}
    stalls = {k: v[i] for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("not_issued")}
    with open(os.path.join(PROF, "r02_k_march_lean_raw.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none, one launch of k_march_lean<4, 8, 256> "
                "(256^3 / 64^3, f32; python tools/variant_ab.py 256 4 6, sixth launch)\n")
        f.write("".join(f"{w} {a} {b}\n" for w, (a, b) in vals.items()))
        f.write("# warp stall samples\n")
        f.write("".join(f"{k} {x}\n" for k, x in sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))
                        if float(x or 0) > 0))
    rd = float(vals["dram__bytes_read.sum"][1]) * UNIT[vals["dram__bytes_read.sum"][0]]
    wr = float(vals["dram__bytes_write.sum"][1]) * UNIT[vals["dram__bytes_write.sum"][0]]
    tpath = os.path.join(PROF, "ncu_traffic.json")
    t = json.load(open(tpath))
    t["c3"] = {"kernel": "k_march_lean", "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
               "source": "profiles/r02_k_march_lean_raw.txt"}
    json.dump(t, open(tpath, "w"), indent=2)
    open(os.path.join(PROF, "r02_k_march_lean_details.txt"), "w").write(ncu("-i", rep, "--page", "details"))
    mix = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_mix.py"), rep], capture_output=True,
                         text=True).stdout
    open(os.path.join(PROF, "r02_k_march_lean_mix.txt"), "w").write(mix)
    src = os.path.join(OUT, "src_final.csv")
    open(src, "w").write(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), src, "30"],
                           capture_output=True, text=True).stdout
    open(os.path.join(PROF, "r02_k_march_lean_lines.txt"), "w").write(lines)
    open(os.path.join(PROF, "r02_k_post_details.txt"), "w").write(
        ncu("-i", os.path.join(OUT, "prof_post_final.ncu-rep"), "--page", "details"))
    # launch list
    tot, cnt = collections.defaultdict(float), collections.Counter()
    hdr = None
    for x in csv.reader(open(os.path.join(OUT, "launches_final.csv"))):
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
    with open(os.path.join(PROF, "r02_launches.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 400 python bench.py "
                "--steps 2 --warmup 3 --no-register --no-cpu-full\n# (cold-cache, serialised per-launch "
                "times: compare SHARES, not absolutes); round 2 final\n")
        f.write(f"# {sum(cnt.values())} launches, {T:.1f} us total\n")
        f.write(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'share':>7s} {'us/launch':>10s}\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            f.write(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k] / T * 100:6.1f}% {tot[k] / cnt[k]:10.1f}\n")
    print(open(os.path.join(PROF, "r02_launches.txt")).read())
    print(open(os.path.join(PROF, "r02_k_march_lean_raw.txt")).read())


if __name__ == "__main__":
    main()
