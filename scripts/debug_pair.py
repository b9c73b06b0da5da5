"""Debug helper: run oracle and GPU side by side (lockstep regrids) and report where they differ (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as orc
import paper_2508_05020_b200 as amr
import workloads as W

def report(o, g, tag):
    so, sg = o.get_state(), g.get_state()
    worst = []
    for k in so:
        d = np.abs(so[k] - sg[k])
        if d.max() > 1e-13:
            idx = np.unravel_index(np.argmax(d), d.shape)
            worst.append((float(d.max()), k, tuple(int(x) for x in idx), float(so[k][idx]), float(sg[k][idx])))
    worst.sort(reverse=True)
    print(tag, "npatch diff>1e-13:", len(worst), flush=True)
    for w in worst[:6]:
        print("   ", w, flush=True)
    return len(worst)

name = sys.argv[1] if len(sys.argv) > 1 else "shock_bubble"
if name == "shock_bubble":
    cfg = W.shock_bubble(Nx=128, Ny=64, n=16, levels=3)
elif name == "sb1":
    cfg = W.shock_bubble(Nx=128, Ny=64, n=16, levels=1)
o = orc.Oracle(cfg); g = amr.Mesh(cfg)
fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)
o.set_state(fn); g.set_state(fn)
def regrid():
    fo = o.flags(); fg = g.flags()
    for k in fo:
        if abs(fo[k][0] - fg[k][0]) > 1e-9 * max(fo[k][0], 0.1):
            print("  flag diff", k, fo[k], fg[k])
    ref = [k for k, v in fo.items() if v[1]]; crs = [k for k, v in fo.items() if v[2]]
    o.regrid_with_requests(ref, crs); g.regrid_with_requests(ref, crs)
for _ in range(cfg["levels"] - 1):
    regrid()
    o.set_state(fn); g.set_state(fn)
report(o, g, "init")
for s in range(1, 9):
    o.step(cfl=0.5); g.step(cfl=0.5)
    report(o, g, f"step {s}")
    if s % 4 == 0:
        regrid(); report(o, g, f"regrid {s}")
