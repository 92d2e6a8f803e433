"""Summarise an ncu source page (CSV from `ncu -i X --page source --csv --print-source cuda,sass`)
per CUDA source line: executed warp instructions, stall samples and top stall reasons.

    python tools/ncu_lines.py report.csv [top]
"""

import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    fname = None
    header = None
    per = defaultdict(lambda: [0, 0, defaultdict(int), ""])
    tot_inst = tot_samp = 0
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            header = r
            continue
        if header is None or r[0] == "" or r[0] == "Function Name":
            continue
        d = dict(zip(header, r))
        try:
            inst = int(d.get("Instructions Executed", "0") or 0)
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        e = per[key]
        e[0] += inst
        e[1] += samp
        e[3] = r[1][:90]
        for h, v in d.items():
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    e[2][h[6:]] += int(v or 0)
                except ValueError:
                    pass
        tot_inst += inst
        tot_samp += samp
    print(f"total warp instructions {tot_inst:,}  stall samples {tot_samp:,}")
    print("by instructions:")
    for (f, ln), (inst, samp, st, src) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        tops = ",".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{f}:{ln:<5d} inst {100 * inst / max(tot_inst, 1):5.1f}%  samp {100 * samp / max(tot_samp, 1):5.1f}%  "
              f"[{tops}]  {src}")
    print("by stall samples:")
    for (f, ln), (inst, samp, st, src) in sorted(per.items(), key=lambda kv: -kv[1][1])[:top // 2]:
        tops = ",".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{f}:{ln:<5d} samp {100 * samp / max(tot_samp, 1):5.1f}%  inst {100 * inst / max(tot_inst, 1):5.1f}%  "
              f"[{tops}]  {src}")


if __name__ == "__main__":
    main()
