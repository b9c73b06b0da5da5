#!/bin/bash
# ncu --set full of the Central4 block-tile kernels (n = 16, 8) and of the AMR auxiliary kernels on configs[3]
# (separate launches: AMR_POST_FUSE=0), for the kernel-level evidence.  Usage: scripts/profile_aux_r2.sh TAG
TAG=${1:-r2}
B="python bench.py --steps 1 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table"
for n in 16 8; do
  ncu --set full --clock-control none --import-source on -k regex:stage_c4_group -s 4 -c 1 -o gpurun_out/c4g${n}_$TAG -f \
      $B --n $n > gpurun_out/ncu_c4g${n}_$TAG.log 2>&1; echo c4g$n $?
done
for k in ghost_tile reflux restrict flags_kernel prolong; do
  AMR_POST_FUSE=0 ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/aux_${k}_$TAG -f \
      python scripts/amr_launches.py sb > gpurun_out/ncu_aux_${k}_$TAG.log 2>&1; echo $k $?
done
ncu --set full --clock-control none -k regex:post_stage -c 1 -o gpurun_out/aux_post_$TAG -f \
    python scripts/amr_launches.py sb > gpurun_out/ncu_aux_post_$TAG.log 2>&1; echo post $?
