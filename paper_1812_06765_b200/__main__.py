"""`python -m paper_1812_06765_b200 ...`: the ngfreg command line on the GPU (cli.py)."""

import sys

from .cli import main

sys.exit(main())
