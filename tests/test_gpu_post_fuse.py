"""The cooperative post-stage kernel (reflux + restriction of every level + the next stage's ghost strips in one
launch, one rank) against the separate reflux / per-level restriction / ghost launches (AMR_POST_FUSE=0): the
same per-cell arithmetic, so the states after AMR steps with regrids must be bitwise equal.  Each variant runs
in its own process (the switch is read once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2508_05020_b200 as amr, workloads as W
case, out = sys.argv[2], sys.argv[3]
cfgs = {
    "quadrant": W.quadrant(N=64, n=16, levels=3, seed=2),
    "shock_bubble": W.shock_bubble(Nx=128, Ny=64, n=16, levels=4),
    "implosion_c4": W.implosion(N=256, n=32, scheme="central4", levels=3, theta=0.05),
    "blast_n8": dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(64, 64), n=8, levels=3, bc=("periodic",) * 4, scheme="weno5",
                     characteristic=1, div_order=4, ic="blast", blast_width=0.08, theta=0.02, coarsen_frac=0.25,
                     weno_eps=1e-6, gamma=1.4),
}
cfg = cfgs[case]
g = amr.Mesh(cfg)
fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)
g.set_state(fn)
for _ in range(cfg["levels"] - 1):
    g.regrid(); g.set_state(fn)
dts = []
for s in range(1, 11):
    dts.append(g.step(cfl=0.45))
    if s % 4 == 0:
        g.regrid()
st = g.stats()
np.savez(out, U=g.get_state(as_dict=False), dts=np.array(dts), keys=np.array(g.keys()), launches=st["launches"])
'''


@pytest.mark.parametrize("case", ["quadrant", "shock_bubble", "implosion_c4", "blast_n8"])
def test_post_stage_fusion_is_bitwise_the_separate_launches(case, tmp_path):
    res = {}
    for fuse in ("1", "0"):
        out = str(tmp_path / f"{case}_{fuse}.npz")
        env = dict(os.environ, AMR_POST_FUSE=fuse)
        r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, case, out], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[fuse] = np.load(out)
    a, b = res["1"], res["0"]
    assert np.array_equal(a["keys"], b["keys"])
    assert np.array_equal(a["dts"], b["dts"])
    assert np.array_equal(a["U"], b["U"])
    assert int(a["launches"]) < int(b["launches"])
