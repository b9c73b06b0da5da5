#!/bin/bash
# A/B of two prebuilt libraries (abso/A.so, abso/B.so) on the AMR extras of bench.py: scripts/ab_so_amr.sh [reps]
R=${1:-2}
SO=paper_2508_05020_b200/libamr.so
for i in $(seq $R); do for v in A B; do
cp abso/$v.so $SO
timeout 600 python bench.py --steps 3 --warmup 3 --no-weno --no-sweep-table --no-cpu-baseline > /tmp/o.json 2>/tmp/e.log
python -c "
import json; d=json.loads([l for l in open('/tmp/o.json') if l.startswith('{')][-1])
print('$v', ' '.join('%s %.3f (stepping %.3f, regrid %.3f)' % (k[:12], d[k]['ms_per_step'], d[k]['step_ms_without_regrid'], d[k]['regrid_ms_per_call']) for k in ('quadrant_amr', 'shock_bubble_amr', 'shock_bubble_amr_subcycled')))" || tail -3 /tmp/e.log
done; done
cp abso/B.so $SO
