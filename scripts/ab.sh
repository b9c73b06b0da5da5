#!/bin/bash
# A/B of the Central4 stage kernel variants in one process environment: scripts/ab.sh [reps]
R=${1:-2}
for i in $(seq $R); do for v in 0 1; do
python bench.py --steps 10 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table --stage-kernel $v > /tmp/o.json 2>/tmp/e.log
python -c "import json; d=json.load(open('/tmp/o.json')); print('variant $v', round(d['roofline']['avg_launch_ms'],4), 'ms', round(d['roofline']['frac'],3))" || tail -3 /tmp/e.log
done; done
nvidia-smi --query-gpu=name,serial,clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv
