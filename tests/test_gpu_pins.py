"""The pinned special cases of tests/test_oracle_dt_flags_reflux.py run through the CUDA path (C ABI):

- the A32 ambiguity band: the GPU's flag kernel must raise the ambiguity bit exactly where the exact
  (rational) indicator lies within 1e-9 of theta or theta/4, and take the strict refine / coarsen decisions
  outside it;
- O13 Lambda (device reduction, amr_diagnostics) against the brute-force maximum over the primitives on a
  3-level mesh, and its NaN stickiness (a NaN cell anywhere makes a CFL step fail without committing).
"""
import math

import numpy as np
import pytest

import oracle as orc
import paper_2508_05020_b200 as amr
import workloads as W
from tests.test_oracle_dt_flags_reflux import build_ramp, expected_flags, ramp_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["refine", "coarsen"])
@pytest.mark.parametrize("delta", [5e-10, -5e-10, 5e-9, -5e-9])
def test_gpu_ambiguity_band(kind, delta):
    cfg, state, rho, lev = ramp_case(kind, delta)
    exp = expected_flags(kind, rho, lev)
    g = amr.Mesh(cfg)
    build_ramp(g, kind, state)
    fl = g.flags()
    o = orc.Oracle(cfg)
    build_ramp(o, kind, state)
    fo = o.flags()
    for P in range(4):
        me, rf, cf, am = fl[(0, P, 0)]
        dec, amb = exp[P]
        assert am == amb, (P, me, am, amb)
        assert (rf if kind == "refine" else cf) == dec, (P, me, dec)
        assert abs(me - fo[(0, P, 0)][0]) <= 1e-14 * abs(fo[(0, P, 0)][0])
    g.close()


def _three_level(scheme="weno5"):
    cfg = dict(lo=(0.0, 0.0), hi=(2.0, 1.0), base=(32, 16), n=8, levels=3, bc=("periodic",) * 4, scheme=scheme,
               characteristic=1, div_order=4, ic="uniform", uniform_state=(1.0, 0.0, 0.0, 1.0))
    g = amr.Mesh(cfg)
    g.regrid_with_requests([(0, 1, 0), (0, 2, 1)])
    g.regrid_with_requests([(1, 3, 1)])
    return cfg, g


@pytest.mark.parametrize("fast_level", [0, 1, 2])
def test_gpu_lambda_brute_force_on_three_levels(fast_level):
    cfg, g = _three_level()
    n = cfg["n"]
    rng = np.random.default_rng(11 + fast_level)
    tr = g.tree()
    U = np.empty((len(tr), 4, n, n))
    lam_bf = 0.0
    for e, d in enumerate(tr):
        rho = rng.uniform(0.5, 2.0, (n, n))
        p = rng.uniform(0.5, 2.0, (n, n))
        boost = 6.0 if d.level == fast_level else 1.0
        u = boost * rng.uniform(-1, 1, (n, n))
        v = boost * rng.uniform(-1, 1, (n, n))
        U[e] = W.to_conserved(rho, u, v, p)
        if d.leaf:
            dx, dy = 2.0 / (32 << d.level), 1.0 / (16 << d.level)
            c = np.sqrt(1.4 * p / rho)
            lam_bf = max(lam_bf, ((np.abs(u) + c) / dx + (np.abs(v) + c) / dy).max())
    g.set_state(U=U)
    # set_state restricts non-leaf patches; Lambda reads leaves only, so the brute force above stands
    _, lam = g.diagnostics()
    assert lam == pytest.approx(lam_bf, rel=1e-13)
    g.close()


def test_gpu_lambda_nan_fails_the_cfl_step_without_commit():
    cfg, g = _three_level()
    g.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    tr = g.tree()
    leaves = [e for e, d in enumerate(tr) if d.leaf]
    e = leaves[len(leaves) // 2]
    U = g.get_state(as_dict=False, indices=np.array([e], np.int32))
    U[0, 3, 2, 3] = -1.0
    g.set_state(U=U, indices=np.array([e], np.int32))
    before = g.get_state(as_dict=False)
    _, lam = g.diagnostics()
    assert math.isnan(lam)
    with pytest.raises(amr.AmrError):
        g.step(cfl=0.5)
    after = g.get_state(as_dict=False)
    assert np.array_equal(before, after, equal_nan=True)
    g.close()
