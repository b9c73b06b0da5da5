"""Stage-kernel time (library CUDA events) on a smooth workload: the isentropic vortex at 4096^2, 32^2 patches,
WENO5-char unless argv[1] == 'central4'.  python scripts/time_stage.py [scheme] (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_05020_b200 as amr  # noqa: E402
import workloads as W  # noqa: E402

scheme = sys.argv[1] if len(sys.argv) > 1 else "weno5"
cfg = W.vortex(N=4096, n=32, scheme=scheme)
g = amr.Mesh(cfg)
g.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
g.steps(2, cfl=0.5)
g.sync()
g.reset_stats()
g.set_kernel_timing(True)
g.steps(5, cfl=0.5)
g.sync()
st = g.stats()
print(scheme, "stage ms %.4f" % (st["stage_ms"] / st["stage_timed"]))
