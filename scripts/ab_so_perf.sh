#!/bin/bash
# A/B of prebuilt libraries abso/<name>.so with scripts/quick_perf.py (args after the names): 
#   scripts/ab_so_perf.sh "A B" sweep amr n=16
NAMES=$1; shift
SO=paper_2508_05020_b200/libamr.so
cp $SO /tmp/libamr_orig.so
for r in 1 2; do for v in $NAMES; do
  cp abso/$v.so $SO
  echo "== $v (rep $r)"
  AMR_NO_BUILD=1 timeout 600 python scripts/quick_perf.py "$@" 2>&1 | tail -12
done; done
cp /tmp/libamr_orig.so $SO
