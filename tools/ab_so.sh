#!/bin/bash
# A/B two builds of the library on the GPU box: tools/ab_so.sh <alt.so> <reps> -- <command>
# alternates the in-tree libngfb200.so (A) with <alt.so> (B) and runs <command> on each.
alt=$1; reps=$2; shift 3
lib=paper_1812_06765_b200/libngfb200.so
cp $lib /tmp/ab_A.so
for r in $(seq $reps); do
  cp /tmp/ab_A.so $lib; echo "== A ($r)"; "$@"
  cp $alt $lib; echo "== B ($r)"; "$@"
done
cp /tmp/ab_A.so $lib
