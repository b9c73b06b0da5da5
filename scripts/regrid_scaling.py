"""Replicated host regrid work per rank at the D4w weak-scaling tree sizes (CPU only, include/amr_debug.h):
a shock-bubble-like refinement (planar shock band at x = 0.2, one bubble ring of radius 0.2 per copy k at
(0.6, k + 0.5), refined to level 3 in bands two patches wide) on the 2048 x 1024 G base of configs[3], G copies
for G ranks; amr_plan_profile times the per-rank plan phases on this machine (max over ranks).

    python scripts/regrid_scaling.py [G ...]
"""
import ctypes as C
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_05020_b200 as amr  # noqa: E402
import workloads as W  # noqa: E402
from tests.test_multirank_host import Plan  # noqa: E402


def build(G):
    cfg = W.shock_bubble(G=G, max_patches=100_000 * G)
    p = Plan(cfg)
    L = p.L
    L.amr_plan_profile.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int64)]
    n, nx0 = 16, 2048
    for lev in range(3):
        tr = p.tree(1)
        h = 2.0 / (nx0 << lev)          # cell size at this level
        w = 2 * n * h                   # band half-width: two patches
        keys = []
        for d in tr:
            if not d.leaf or d.level != lev:
                continue
            x0, y0 = d.i * n * h, d.j * n * h
            xc, yc = x0 + 0.5 * n * h, y0 + 0.5 * n * h
            k = min(int(yc), G - 1)
            r = math.hypot(xc - 0.6, yc - (k + 0.5))
            if abs(xc - 0.2) < w or abs(r - 0.2) < w:
                keys.append((d.level, d.i, d.j))
        p.refine(keys)
    return p


def main():
    Gs = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
    out = {}
    for G in Gs:
        p = build(G)
        worst = None
        for r in range(G):
            ms = (C.c_double * 7)()
            cnt = (C.c_int64 * 4)()
            assert p.L.amr_plan_profile(p.h, G, r, 3, ms, cnt) == 0
            row = {"ms": [round(x, 3) for x in ms], "patches": cnt[0], "leaves": cnt[1], "halo_recv_items": cnt[2],
                   "halo_send_items": cnt[3]}
            if worst is None or ms[6] > worst["ms"][6]:
                worst = row
        out[G] = worst
        print(json.dumps({"G": G, **worst}), flush=True)
    return out


if __name__ == "__main__":
    main()
