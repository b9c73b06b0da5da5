#!/bin/bash
# ncu --set full of one stage-2 launch of the fused Central4 kernel on the sweep; usage: scripts/gpu_prof.sh TAG [regex] [bench args]
TAG=${1:-p}; RX=${2:-stage_c4}; shift; shift
ncu --set full --clock-control none --import-source on -k regex:$RX -s 4 -c 1 -o gpurun_out/$TAG -f \
    python bench.py --steps 1 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table "$@" > gpurun_out/ncu_$TAG.log 2>&1; echo ncu $?
