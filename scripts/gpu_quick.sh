#!/bin/bash
# quick GPU check: Central4 parity subset + sweep bench (no extras); usage: scripts/gpu_quick.sh TAG [bench args]
TAG=${1:-q}; shift
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "central4 or variants or vortex or patch_size" > gpurun_out/t_$TAG.log 2>&1; echo tests $?; tail -3 gpurun_out/t_$TAG.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table "$@" > gpurun_out/b_$TAG.log 2>&1; echo bench $?
python - <<PY
import json
l=[x for x in open("gpurun_out/b_$TAG.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); r=d["roofline"]
    print("value %.3e  launch %.4f ms  frac %.3f  clocks %s" % (d["value"], r["avg_launch_ms"], r["frac"], d["clocks"]))
else:
    print(open("gpurun_out/b_$TAG.log").read()[-2000:])
PY
