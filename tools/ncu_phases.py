"""Split the fused march's executed instructions by phase from an ncu source-page export.

    python tools/ncu_phases.py gpurun_out/src_<tag>.csv > profiles/r01_k_eval_fused_<tag>_phases.txt

The export (`ncu -i prof.ncu-rep --page source --csv --print-source sass`, written by
tools/profiles_refresh.py) lists every SASS instruction under the source line it came
from.  Instructions of inlined helpers (fused_impl.cuh, cmath) are charged to the
fused_march.cuh line that precedes them in address order, and fused_march.cuh lines are
mapped to phases by the section markers in the source itself, so the split follows the
code as compiled for that capture.
"""

import collections
import csv
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1812_06765_b200", "csrc", "fused_march.cuh")


def phase_table():
    """(first line, phase) pairs from the markers in fused_march.cuh, in line order."""
    marks = [
        (r"void load_yplane\(", "A: P_xy y of a new deformation plane (load_yplane)"),
        (r"^// Reduce a completed deformation plane", "flush: x/y P^T reduction of a finished def plane"),
        (r"^// One axis of the template cell lookup", "A: cell lookup (cell_axis)"),
        (r"void fused_step\(", "step control"),
        (r"-{10,} \(A\) plane p", "A: yhat, 8-corner gathers, W and dT/h"),
        (r"-{10,} \(B\) q on plane", "B: grad W, NGF ratio, D, q"),
        (r"-{10,} \(C\) s, ghat", "C: G^T, warp Jacobian^T, z-P^T accumulation"),
        (r"const int zdj = sm\.zi", "flush: x/y P^T reduction of a finished def plane"),
        (r"^// CTA geometry of the march", "CTA setup (tables, slot geometry)"),
        (r"k_eval_fused\(const __grid_constant__", "march loop / CTA setup"),
    ]
    lines = open(SRC).read().splitlines()
    out = []
    for pat, name in marks:
        for i, l in enumerate(lines, 1):
            if re.search(pat, l):
                out.append((i, name))
                break
    return sorted(out)


def main():
    table = phase_table()

    def phase(line):
        name = "other"
        for first, n in table:
            if line >= first:
                name = n
        return name

    rows = list(csv.reader(open(sys.argv[1])))
    ins = []
    cur_file, cur_line = None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0]:
            cur_line = int(r[0])
            continue
        if r[2].startswith("0x"):
            try:
                n = int(r[7])
            except ValueError:
                n = 0
            sass = r[3].split()
            op = sass[1] if sass and sass[0].startswith("@") and len(sass) > 1 else (sass[0] if sass else "")
            ins.append((int(r[2], 16), cur_file, cur_line, op.split(".")[0], n))
    ins.sort()
    agg, ops = collections.Counter(), collections.defaultdict(collections.Counter)
    cur = "march loop / CTA setup"
    for _, f, line, op, n in ins:
        if f == "fused_march.cuh":
            cur = phase(line)
        agg[cur] += n
        ops[cur][op] += n
    tot = sum(agg.values())
    print(f"k_eval_fused warp instructions executed by phase ({sys.argv[1]}), total {tot / 1e6:.1f} M")
    for p, n in agg.most_common():
        top = ", ".join(f"{o} {c / 1e6:.1f}" for o, c in ops[p].most_common(8))
        print(f"{100 * n / tot:5.1f} %  {n / 1e6:6.1f} M  {p:50s}  [{top}]")


if __name__ == "__main__":
    main()
