cd $GRAFT_REPO_ROOT
AMR_NVCC_FLAGS=-DAMR_PHASE_PROF python -m paper_2508_05020_b200.build > gpurun_out/pbuild.log 2>&1 || echo buildfail
for n in 8 16 32; do
AMR_NO_BUILD=1 AMR_PHASE_PROF=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table --n $n > gpurun_out/p$n.json 2> gpurun_out/p$n.err
echo n=$n; grep -A4 'stage 2' gpurun_out/p$n.err | tail -5
done
python -m paper_2508_05020_b200.build > /dev/null 2>&1
for n in 8 16; do timeout 300 python bench.py --steps 10 --warmup 3 --no-weno --no-amr --no-cpu-baseline --no-sweep-table --n $n > /tmp/o.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/o.json')); print('n=$n', round(d['roofline']['avg_launch_ms'],4), 'ms', round(d['roofline']['frac'],3))"; done
