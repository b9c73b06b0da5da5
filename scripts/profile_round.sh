#!/bin/bash
# Round-end evidence set (GPU box): default bench line, the launch list of the headline bench command, ncu --set full
# of the stage kernels (profile_r2.sh) and of the block-tile / AMR auxiliary kernels (profile_aux_r2.sh), and the
# AMR per-kernel launch breakdown (amr_launches.py under ncu).  Usage: scripts/profile_round.sh TAG
TAG=${1:-r2f}
cd ${GRAFT_REPO_ROOT:-.}
python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-amr --no-sweep-table > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches $?
bash scripts/profile_r2.sh $TAG
bash scripts/profile_aux_r2.sh $TAG
bash scripts/amr_profile.sh $TAG
