"""Import the unmodified reference package staged by oracle/build_ref.py (test infrastructure).

`load()` returns the `ngfreg` module from oracle/_ref (or from /root/reference in the
build container), or None when neither exists.  Only tests/, smoke() and bench.py's
CPU legs call this; the product package never does.
"""

from __future__ import annotations

import importlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CANDIDATES = (os.path.join(HERE, "_ref"), "/root/reference/pkg/src")


def load():
    for root in CANDIDATES:
        if os.path.isfile(os.path.join(root, "ngfreg", "__init__.py")):
            if root not in sys.path:
                sys.path.insert(0, root)
            sys.dont_write_bytecode = True
            return importlib.import_module("ngfreg")
    return None


def origin() -> str:
    m = load()
    return "none" if m is None else os.path.dirname(os.path.dirname(m.__file__))
