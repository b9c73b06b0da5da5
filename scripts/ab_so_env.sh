#!/bin/bash
# A/B of prebuilt libraries with per-variant environment: scripts/ab_so_env.sh "name:VAR=val,VAR2=val name2:" <quick_perf args>
# (name = abso/<name>.so; the part after ':' is a comma-separated environment for that variant)
VARS=$1; shift
SO=paper_2508_05020_b200/libamr.so
cp $SO /tmp/libamr_orig.so
for r in 1 2; do for v in $VARS; do
  name=${v%%:*}; envs=${v#*:}
  cp abso/$name.so $SO
  echo "== $v (rep $r)"
  env ${envs//,/ } AMR_NO_BUILD=1 timeout 600 python scripts/quick_perf.py "$@" 2>&1 | tail -12
done; done
cp /tmp/libamr_orig.so $SO
