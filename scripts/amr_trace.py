"""Launch timeline of AMR steps (GPU box): AMR_TRACE=<file> python scripts/amr_trace.py q|sb [K]
Runs the init protocol, 8 warm-up steps with 2 regrids, then K steps (regrid every 4); the library appends
"name start_us duration_us" per launch to <file> at close; this script then prints the last K steps' timeline
summary: per launch kind total device time, and the gaps between launches."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_05020_b200 as amr  # noqa: E402
import workloads as W  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "q"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = (W.shock_bubble(max_patches=100_000) if which in ("sb", "sbs") else W.quadrant(N=512, n=16, levels=3, seed=1))
if which == "sbs":   # with Berger-Colella subcycling
    cfg["subcycle"] = 1
out = os.environ["AMR_TRACE"]
if os.path.exists(out):
    os.remove(out)
g = amr.Mesh(cfg)
fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
g.set_state(fn)
for _ in range(cfg["levels"] - 1):
    g.regrid()
    g.set_state(fn)
for s in range(1, 9):
    g.step(cfl=0.5)
    if s % 4 == 0:
        g.regrid()
for s in range(1, K + 1):
    g.step(cfl=0.5)
    if s % 4 == 0:
        g.regrid()
g.close()
rows = [l.split() for l in open(out)]
rows = [(r[0] if len(r) == 3 else " ".join(r[:-2]), float(r[-2]), float(r[-1])) for r in rows]
dts = [i for i, r in enumerate(rows) if r[0] == "dt"]
first = dts[-K]
seg = rows[first:]
t0 = seg[0][1]
t1 = seg[-1][1] + seg[-1][2]
agg = defaultdict(lambda: [0, 0.0])
gap = 0.0
prev_end = t0
big = []
for name, st, du in seg:
    agg[name][0] += 1
    agg[name][1] += du
    gp = st - prev_end
    gap += max(0.0, gp)
    if gp > 20:
        big.append((name, round(gp, 1)))
    prev_end = st + du
span = t1 - t0
print(f"{which}: {K} steps, span {span:.1f} us = {span / K:.1f} us/step; launches {len(seg)}; gaps {gap:.1f} us "
      f"({gap / K:.1f} us/step)")
for k, (n, tt) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:14s} n={n:4d} total {tt:9.1f} us  mean {tt / n:7.2f} us  per step {tt / K:8.1f} us")
print("  gaps > 20 us before:", big[:20])
