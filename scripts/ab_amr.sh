#!/bin/bash
# A/B of two builds on the AMR extras of bench.py (quadrant, shock-bubble, subcycled): scripts/ab_amr.sh "<flags A>" "<flags B>" [reps]
FA=$1; FB=$2; R=${3:-2}
SO=paper_2508_05020_b200/libamr.so
AMR_NVCC_FLAGS="$FA" python -m paper_2508_05020_b200.build > /dev/null 2>&1 && cp $SO /tmp/A.so || echo "build A failed"
AMR_NVCC_FLAGS="$FB" python -m paper_2508_05020_b200.build > /dev/null 2>&1 && cp $SO /tmp/B.so || echo "build B failed"
for i in $(seq $R); do for v in A B; do
cp /tmp/$v.so $SO
timeout 600 python bench.py --steps 3 --warmup 3 --no-weno --no-sweep-table --no-cpu-baseline > /tmp/o.json 2>/tmp/e.log
python -c "
import json; d=json.loads([l for l in open('/tmp/o.json') if l.startswith('{')][-1])
print('$v', ' '.join('%s %.3f (stepping %.3f)' % (k[:12], d[k]['ms_per_step'], d[k]['step_ms_without_regrid']) for k in ('quadrant_amr', 'shock_bubble_amr', 'shock_bubble_amr_subcycled')))" || tail -3 /tmp/e.log
done; done
cp /tmp/B.so $SO
