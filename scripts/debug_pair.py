"""Debug helper: run oracle and GPU side by side and report where they differ (GPU box)."""
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
        if d.max() > 0:
            idx = np.unravel_index(np.argmax(d), d.shape)
            worst.append((d.max(), k, idx, so[k][idx], sg[k][idx]))
    worst.sort(reverse=True)
    print(tag, "npatch diff", len(worst))
    for w in worst[:8]:
        print("   ", w)

cfg = W.shock_bubble(Nx=128, Ny=64, n=16, levels=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
o = orc.Oracle(cfg); g = amr.Mesh(cfg)
fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)
o.set_state(fn); g.set_state(fn)
for _ in range(cfg["levels"] - 1):
    fo = o.flags()
    ref = [k for k, v in fo.items() if v[1]]; crs = [k for k, v in fo.items() if v[2]]
    o.regrid_with_requests(ref, crs); g.regrid_with_requests(ref, crs)
    o.set_state(fn); g.set_state(fn)
report(o, g, "init")
for s in range(3):
    o.step(cfl=0.5); g.step(cfl=0.5)
    report(o, g, f"step {s+1}")
