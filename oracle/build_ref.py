"""Recipe: stage the UNMODIFIED reference package into oracle/_ref (test infrastructure).

    python oracle/build_ref.py            # run by __graft_entry__.build() when /root/reference exists

The reference (`ngfreg`, /root/reference/pkg/src/ngfreg) is pure Python + numpy, so
"building" it is copying its source files, byte for byte, into oracle/_ref/ngfreg.
oracle/_ref is git-ignored (the reference source never enters this repository's
history) but not gpurun-ignored, so it travels to the GPU box, where /root/reference
does not exist.  Only the checker and the baseline legs use it: tests/, smoke(),
bench.py's cpu_baseline / --impl reference.  The product package never imports it.
A STAMP file records the SHA-256 of every staged file.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import sys

SRC = "/root/reference/pkg/src/ngfreg"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "_ref", "ngfreg")


def main() -> int:
    if not os.path.isdir(SRC):
        print(f"build_ref: {SRC} absent; keeping {DST} as staged" if os.path.isdir(DST)
              else f"build_ref: {SRC} absent and nothing staged")
        return 0
    os.makedirs(DST, exist_ok=True)
    stamp = []
    for name in sorted(os.listdir(SRC)):
        if not name.endswith(".py"):
            continue
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
        with open(os.path.join(DST, name), "rb") as fh:
            stamp.append(f"{hashlib.sha256(fh.read()).hexdigest()}  {name}")
    with open(os.path.join(HERE, "_ref", "STAMP"), "w") as fh:
        fh.write("\n".join(stamp) + "\n")
    print(f"build_ref: staged {len(stamp)} files of ngfreg into {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
