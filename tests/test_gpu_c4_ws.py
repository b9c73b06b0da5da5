"""The warp-specialised Central4 kernel (stage_c4_ws_kernel: face passes of tile k overlapped with the conversion of
tile k+1 and the epilogue of tile k-1) against the phase-serial per-tile TMA kernel: the same per-cell arithmetic, so
bitwise equal states on the 32^2 / 64^2 paths (uniform noise sweep, AMR implosion with regrids and C/F faces,
subcycled covered patches).  Each kernel runs in its own process (AMR_C4_WS, read once per process)."""
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
    "noise_n32": dict(W.sweep(N=512, n=32, scheme="central4", seed=7), check_positivity=0),
    "noise_n64": dict(W.sweep(N=512, n=64, scheme="central4", seed=7), check_positivity=0),
    "implosion_amr_n32": W.implosion(N=256, n=32, scheme="central4", levels=3, theta=0.05),
    "vortex_walls_subcycled_n32": dict(W.vortex(N=128, n=32, levels=2, theta=0.01,
                                                bc=("transmissive", "transmissive", "reflective", "reflective")), subcycle=1),
}
cfg = cfgs[case]
g = amr.Mesh(cfg)
fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)
g.set_state(fn)
for _ in range(cfg["levels"] - 1):
    g.regrid(); g.set_state(fn)
_, lam = g.diagnostics()
for s in range(1, 7):
    if cfg.get("check_positivity", 1):
        g.step(cfl=0.4)
    else:
        g.step(dt=0.3 / lam)
    if cfg["levels"] > 1 and s % 3 == 0:
        g.regrid()
np.savez(out, U=g.get_state(as_dict=False), keys=np.array(g.keys()))
'''


@pytest.mark.parametrize("case", ["noise_n32", "noise_n64", "implosion_amr_n32", "vortex_walls_subcycled_n32"])
def test_warp_specialised_kernel_is_bitwise_the_per_tile_kernel(case, tmp_path):
    res = {}
    for ws in ("1", "0"):
        out = str(tmp_path / f"{case}_{ws}.npz")
        env = dict(os.environ, AMR_C4_WS=ws)
        r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, case, out], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-3000:]
        res[ws] = np.load(out)
    assert np.array_equal(res["1"]["keys"], res["0"]["keys"])
    assert np.array_equal(res["1"]["U"], res["0"]["U"], equal_nan=True)
