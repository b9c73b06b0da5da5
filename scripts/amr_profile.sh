#!/bin/bash
# AMR step evidence (GPU box): per-kernel launch list of 4 steps + 1 regrid of configs[2] and configs[3] under ncu,
# the host regrid phase timers, and the step / regrid times with and without CUDA graphs.  TAG names the outputs.
TAG=${1:-r2}
for w in q sb; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/amr_launches_${w}_$TAG.csv \
      python scripts/amr_launches.py $w > gpurun_out/amr_launches_${w}_$TAG.log 2>&1; echo launches $w $?
done
AMR_REGRID_PROF=1 python scripts/amr_launches.py sb > gpurun_out/amr_regrid_prof_sb_$TAG.log 2>&1; echo regrid_prof $?
python scripts/quick_perf.py amr amr_graphs > gpurun_out/amr_perf_$TAG.log 2>&1; echo perf $?
