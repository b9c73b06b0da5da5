#!/bin/bash
# Round profile set: bench line, launch list (gpu__time_duration per launch), ncu --set full of the Central4 and
# WENO stage kernels (stage 2 of step 2).  Usage: scripts/gpu_round_profile.sh TAG
TAG=${1:-r1}
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo bench $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-amr > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches $?
ncu --set full --clock-control none --import-source on -k regex:stage_c4 -s 4 -c 1 -o gpurun_out/c4_$TAG -f \
    python bench.py --steps 1 --warmup 3 --no-weno --no-amr --no-cpu-baseline > gpurun_out/ncu_c4_$TAG.log 2>&1; echo c4 $?
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 4 -c 1 -o gpurun_out/weno_$TAG -f \
    python bench.py --steps 1 --warmup 3 --scheme weno5 --no-weno --no-amr --no-cpu-baseline > gpurun_out/ncu_weno_$TAG.log 2>&1; echo weno $?
