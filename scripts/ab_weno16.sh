#!/bin/bash
# A/B of two builds on the WENO n = 16 paths (AMR configs' stage kernel + uniform sweep): scripts/ab_weno16.sh "<flags A>" "<flags B>"
cd $GRAFT_REPO_ROOT
SO=paper_2508_05020_b200/libamr.so
AMR_NVCC_FLAGS="$1" python -m paper_2508_05020_b200.build > /dev/null 2>&1 && cp $SO /tmp/A.so
AMR_NVCC_FLAGS="$2" python -m paper_2508_05020_b200.build > /dev/null 2>&1 && cp $SO /tmp/B.so
for i in 1 2; do for v in A B; do
cp /tmp/$v.so $SO
echo "== $v"; python scripts/amr_ab_variant.py 2>&1 | grep 'stage_kernel 0' | sort -u
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-sweep-table --no-amr --no-weno --n 16 --scheme weno5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sweep n16 weno', d['roofline']['avg_launch_ms'])"
done; done
cp /tmp/B.so $SO
