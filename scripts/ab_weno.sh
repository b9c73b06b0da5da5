#!/bin/bash
# WENO5-char stage timing at n = 32 and n = 16 (4096^2 sweep) + quadrant AMR step; usage: scripts/ab_weno.sh TAG
for n in 32 16; do
python bench.py --steps 4 --warmup 2 --scheme weno5 --n $n --no-weno --no-amr --no-cpu-baseline --no-sweep-table > /tmp/o.json 2>/tmp/e.log
python -c "import json; d=json.load(open('/tmp/o.json')); print('$1 weno n=$n', round(d['roofline']['avg_launch_ms'],4), 'ms', round(d['value']/1e9,3), 'G')" || tail -3 /tmp/e.log
done
