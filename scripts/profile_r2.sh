#!/bin/bash
# ncu --set full captures of the stage kernels (stage 2 of step 2 of bench's sweep workload) for the kernel-level
# evidence and the fp64 SASS work per cell-stage: Central4 TMA n = 32 (headline), WENO5-char n = 16 (the AMR
# configs' patch size), n = 32, and the n = 8 block-tile kernel.  Usage: scripts/profile_r2.sh TAG
TAG=${1:-r2}
B="python bench.py --steps 1 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table"
ncu --set full --clock-control none --import-source on -k regex:stage_c4_tma -s 4 -c 1 -o gpurun_out/c4_$TAG -f \
    $B > gpurun_out/ncu_c4_$TAG.log 2>&1; echo c4 $?
for n in 16 32; do
  ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 4 -c 1 -o gpurun_out/weno${n}_$TAG -f \
      $B --scheme weno5 --n $n > gpurun_out/ncu_weno${n}_$TAG.log 2>&1; echo weno$n $?
done
ncu --set full --clock-control none --import-source on -k regex:stage_group_kernel -s 4 -c 1 -o gpurun_out/weno8_$TAG -f \
    $B --scheme weno5 --n 8 > gpurun_out/ncu_weno8_$TAG.log 2>&1; echo weno8 $?
