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
# post-process on the box (the full reports exceed what gpurun brings back): summaries, fp64 work, the Central4
# source page; keep only the Central4 and WENO n = 16 reports
C=16777216
python scripts/profile_summary.py $TAG gpurun_out/c4_$TAG.ncu-rep gpurun_out/weno16_$TAG.ncu-rep \
    gpurun_out/weno32_$TAG.ncu-rep gpurun_out/weno8_$TAG.ncu-rep gpurun_out/c4g16_$TAG.ncu-rep gpurun_out/c4g8_$TAG.ncu-rep \
    gpurun_out/aux_post_$TAG.ncu-rep gpurun_out/aux_ghost_tile_$TAG.ncu-rep gpurun_out/aux_reflux_$TAG.ncu-rep \
    gpurun_out/aux_restrict_$TAG.ncu-rep gpurun_out/aux_flags_kernel_$TAG.ncu-rep gpurun_out/aux_prolong_$TAG.ncu-rep \
    > gpurun_out/summary_$TAG.log 2>&1; echo summary $?
cp profiles/${TAG}_ncu_summary.jsonl profiles/${TAG}_launches.json gpurun_out/ 2>/dev/null
python scripts/fp64_work.py gpurun_out/${TAG}_fp64_work.json weno5_char_n16=gpurun_out/weno16_$TAG.ncu-rep:$C \
    weno5_char_n32=gpurun_out/weno32_$TAG.ncu-rep:$C weno5_char_n8=gpurun_out/weno8_$TAG.ncu-rep:$C \
    central4_n32=gpurun_out/c4_$TAG.ncu-rep:$C central4_n16=gpurun_out/c4g16_$TAG.ncu-rep:$C \
    central4_n8=gpurun_out/c4g8_$TAG.ncu-rep:$C > gpurun_out/fp64_$TAG.log 2>&1; echo fp64 $?
ncu -i gpurun_out/c4_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/c4_${TAG}_src.csv 2>/dev/null
for f in gpurun_out/*_$TAG.ncu-rep; do
  case $f in *c4_$TAG.ncu-rep|*weno16_$TAG.ncu-rep) ;; *) rm -f $f ;; esac
done
python scripts/fusion_study.py --N 2048 --warmup 4 --steps 3 --tag $TAG > gpurun_out/fusion_$TAG.log 2>&1; echo fusion $?
cp profiles/${TAG}_fusion_study.json gpurun_out/ 2>/dev/null
du -sh gpurun_out
