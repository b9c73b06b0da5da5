"""Per-kernel time breakdown of AMR steps (run under `ncu --metrics gpu__time_duration.sum`): configs[3]
shock-bubble (or configs[2] quadrant), init protocol, 4 warm-up steps, then 4 steps + 1 regrid profiled.
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv python scripts/amr_launches.py sb
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_05020_b200 as amr  # noqa: E402
import workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "sb"
cfg = W.shock_bubble(max_patches=100_000) if which == "sb" else W.quadrant(N=512, n=16, levels=3, seed=1)
if len(sys.argv) > 2:
    cfg["subcycle"] = int(sys.argv[2])
g = amr.Mesh(cfg)
fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
g.set_state(fn)
for _ in range(cfg["levels"] - 1):
    g.regrid()
    g.set_state(fn)
for s in range(4):
    g.step(cfl=0.5)
g.sync()
print("profiled region", flush=True)
for s in range(4):
    g.step(cfl=0.5)
g.regrid()
g.sync()
st = g.stats()
print({k: st[k] for k in ("leaves", "patches", "proxies", "leaf_cells")})
