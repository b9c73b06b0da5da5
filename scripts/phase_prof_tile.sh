#!/bin/bash
# phase timers of the per-tile Central4 kernel at n = 32 and n = 64 (scripts/phase_prof.sh covers the group kernels)
cd $GRAFT_REPO_ROOT
AMR_NVCC_FLAGS=-DAMR_PHASE_PROF python -m paper_2508_05020_b200.build > gpurun_out/pbuild.log 2>&1 || echo buildfail
for n in 32 64; do
AMR_NO_BUILD=1 AMR_PHASE_PROF=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table --n $n > /dev/null 2> gpurun_out/pt$n.err
echo n=$n; grep -A4 '^stage [123]' gpurun_out/pt$n.err | tail -15
done
python -m paper_2508_05020_b200.build > /dev/null 2>&1
