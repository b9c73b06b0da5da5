"""Plan validation in lieu of compute-sanitizer (closed on this GPU pool): with AMR_CHECK_PLAN=1 every descriptor
index the kernels dereference is checked against the tree and the buffer extents at every plan (DESIGN s6), and with
AMR_CHECK_INCR=1 the incremental leaf order / face-neighbour table against the full rebuild at every regrid.  A
3-level WENO quadrant, a 4-level shock-bubble piece with walls and a Central4 n = 16 block-tile case run with regrids
in a child process with both set; any violation fails the call with AMR_E_STATE."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import paper_2508_05020_b200 as amr, workloads as W
cases = [W.quadrant(N=256, n=16, levels=3, seed=2),
         W.shock_bubble(Nx=256, Ny=128, levels=4, max_patches=20000),
         W.vortex(N=128, n=16, levels=2, theta=0.01, scheme="central4")]
for cfg in cases:
    g = amr.Mesh(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)
    g.set_state(fn)
    for _ in range(cfg["levels"] - 1):
        g.regrid(); g.set_state(fn)
    for s in range(12):
        g.step(cfl=0.4)
        if s % 3 == 2:
            g.regrid()
    g.close()
print("plan checks ok")
"""


@pytest.mark.gpu
def test_plan_and_incremental_checks():
    env = dict(os.environ, AMR_CHECK_PLAN="1", AMR_CHECK_INCR="1")
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0 and "plan checks ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
