#!/bin/bash
# A/B of two prebuilt libraries (abso/A.so, abso/B.so; e.g. two commits): scripts/ab_so.sh [reps] [bench args]
R=${1:-3}; shift
SO=paper_2508_05020_b200/libamr.so
for i in $(seq $R); do for v in A B; do
cp abso/$v.so $SO
timeout 300 python bench.py --steps 10 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table "$@" > /tmp/o.json 2>/tmp/e.log
python -c "import json; d=json.load(open('/tmp/o.json')); print('$v', round(d['roofline']['avg_launch_ms'],4), 'ms', round(d['roofline']['frac'],3), 'step', round(d['ms_per_step'],4))" || tail -3 /tmp/e.log
done; done
cp abso/B.so $SO
