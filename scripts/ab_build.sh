#!/bin/bash
# A/B of two builds of the library on the same box: scripts/ab_build.sh "<flags A>" "<flags B>" [reps] [bench args]
# (flags go to AMR_NVCC_FLAGS; an empty string is the default build)
FA=$1; FB=$2; R=${3:-3}; shift 3
SO=paper_2508_05020_b200/libamr.so
AMR_NVCC_FLAGS="$FA" python -m paper_2508_05020_b200.build > /dev/null 2>&1 && cp $SO /tmp/A.so || echo "build A failed"
AMR_NVCC_FLAGS="$FB" python -m paper_2508_05020_b200.build > /dev/null 2>&1 && cp $SO /tmp/B.so || echo "build B failed"
for i in $(seq $R); do for v in A B; do
cp /tmp/$v.so $SO
timeout 300 python bench.py --steps 10 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table "$@" > /tmp/o.json 2>/tmp/e.log
python -c "import json; d=json.load(open('/tmp/o.json')); print('$v', round(d['roofline']['avg_launch_ms'],4), 'ms', round(d['roofline']['frac'],3), 'step', round(d['ms_per_step'],4))" || tail -3 /tmp/e.log
done; done
cp /tmp/B.so $SO
