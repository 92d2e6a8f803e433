#!/bin/bash
# eval time per forced f32 variant at the pyramid sizes (tools/small_levels.py)
for v in 1 2 4 5; do echo "variant $v"; NGF_FUSED_VARIANT=$v python tools/small_levels.py | sed 's/two_loop.*//'; done
