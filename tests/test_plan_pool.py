"""The regrid's plan phases on the host thread pool (csrc/plan.h: leaf launch order, face-neighbour table, leaf
descriptors with proxy-strip and reflux tasks, computed in parts and merged in part order) give byte for byte the
serial plan -- on the shock-bubble-like D4w tree of scripts/regrid_scaling.py and on random 3-level trees, for one
rank and for the ranks of 2- and 3-way partitions with halo_mode 2.  Host only (include/amr_debug.h)."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/scripts'); sys.path.insert(0, {root!r} + '/tests')
import regrid_scaling as R
from test_multirank_host import Plan, amr_mesh_cfg

def check(p, world, rank, hm):
    L = p.L
    L.amr_plan_build_check.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    ms = (C.c_double * 6)(); cnt = (C.c_int64 * 4)(); eq = C.c_int32()
    assert L.amr_plan_build_check(p.h, world, rank, hm, 2, ms, cnt, C.byref(eq)) == 0
    assert eq.value == 1, (world, rank, hm, list(cnt))
    assert cnt[3] == 4 and cnt[0] > 0
    return list(cnt)

p = R.build(1)
assert check(p, 1, 0, 0)[0] == 20360
for r in range(2):
    check(R.build(2), 2, r, 2)
rng = np.random.default_rng(5)
for trial in range(4):
    p = Plan(amr_mesh_cfg())
    for lev in range(2):
        leaves = [(d.level, d.i, d.j) for d in p.tree(1) if d.leaf and d.level == lev]
        pick = rng.choice(len(leaves), size=max(1, len(leaves) // 5), replace=False)
        p.refine([leaves[k] for k in pick])
    check(p, 1, 0, 0)
    for r in range(3):
        check(p, 3, r, 2)
print("ok")
"""


def test_pooled_plan_equals_serial_plan():
    env = dict(os.environ, AMR_HOST_THREADS="4")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
