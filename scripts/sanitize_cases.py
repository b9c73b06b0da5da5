#!/usr/bin/env python
"""Small end-to-end cases for compute-sanitizer (SURVEY s4 layer 4): every kernel family of the path runs at
least once -- Central4 TMA kernel (n = 32, AMR with C/F faces and walls), Central4 group kernel (n = 16, AMR
blocks + single leaves), WENO5-char (n = 8, 3-level quadrant with regrids: ghost / prolong / reflux / restrict /
flags / Lambda kernels), unfused and per-patch organisations, CUDA-graph replay, the Sod strip."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_05020_b200 as amr  # noqa: E402
import workloads as W  # noqa: E402


def run(cfg, steps=3, regrid_every=2):
    g = amr.Mesh(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    g.set_state(fn)
    for _ in range(cfg["levels"] - 1):
        g.regrid()
        g.set_state(fn)
    for s in range(1, steps + 1):
        g.step(cfl=0.4)
        if regrid_every and s % regrid_every == 0:
            g.regrid()
    g.diagnostics()
    g.close()


cases = [
    dict(W.vortex(N=64, n=32, levels=2, theta=0.01, bc=("transmissive", "transmissive", "reflective", "reflective"))),
    dict(W.vortex(N=64, n=16, levels=2, theta=0.01)),
    dict(W.quadrant(N=32, n=8, levels=3, seed=1)),
    dict(W.quadrant(N=32, n=8, levels=2, seed=2, stage_kernel=2)),
    dict(W.quadrant(N=32, n=8, levels=2, seed=3, stage_kernel=3)),
    dict(W.vortex(N=64, n=32, use_graphs=1)),
    dict(W.sod(), dim=1),
]
for c in cases:
    run(c, steps=5 if c.get("use_graphs") else 3)
print("sanitize cases done")
