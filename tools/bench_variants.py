"""The reference's desk benchmark (ngfreg benchmark, benchmark.py:88-153) on the GPU:
P^T variants cross-checked first, then apply_P / apply_Pt per variant / ngf_value_grad /
register timed per precision.

    python tools/bench_variants.py [--dims 64,64,64] [--precisions f64,f32] [--reps 3] [--out t.tsv]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_06765_b200 import benchmark as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="64,64,64")
    ap.add_argument("--precisions", default="f64,f32")
    ap.add_argument("--variants", default="gather,scatter,redblack")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-iter", type=int, default=10)
    ap.add_argument("--out")
    a = ap.parse_args()
    recs = B.run_benchmark(dims=tuple(int(v) for v in a.dims.split(",")),
                           precisions=tuple(a.precisions.split(",")),
                           variants=tuple(a.variants.split(",")), reps=a.reps,
                           register_max_iter=a.max_iter)
    table = B.format_table(recs)
    print(table)
    if a.out:
        with open(a.out, "w") as f:
            f.write(table + "\n")


if __name__ == "__main__":
    main()
