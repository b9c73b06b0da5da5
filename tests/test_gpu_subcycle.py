"""GPU parity of Berger-Colella time subcycling (NEXT #4, subcycle = 1) against the oracle's subcycled step
(readings S1-S6): every level advanced with its own dt, C/F ghosts interpolated in time, accumulated registers,
reflux and restriction at the common time; trees and flags in lockstep with regrids (A32)."""
import numpy as np
import pytest

import paper_2508_05020_b200 as amr
import workloads as W
from tests.parity import run_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("char", [1, 0])
def test_quadrant_three_levels(char):
    cfg = dict(W.quadrant(N=64, n=16, levels=3, seed=1, characteristic=char), subcycle=1)
    o, g, e = run_pair(cfg, steps=10, cfl=0.5, regrid_every=4)
    assert len({k[0] for k in g.leaves()}) == 3


@pytest.mark.parametrize("n", [32, 8])
def test_central4_two_levels_walls(n):
    """Central4 through the TMA kernel (n = 32) and the per-tile kernel (n = 8) on a 2-level mesh with
    transmissive / reflective walls."""
    N = 128
    cfg = dict(W.vortex(N=N, n=n, levels=2, theta=0.01, bc=("transmissive", "transmissive", "reflective",
                                                            "reflective")), subcycle=1)
    o, g, e = run_pair(cfg, steps=10, cfl=0.5, regrid_every=4)
    assert len({k[0] for k in g.leaves()}) == 2


def test_blast_periodic_three_levels_n8():
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(64, 64), n=8, levels=3, bc=("periodic",) * 4,
               scheme="weno5", characteristic=1, div_order=4, ic="blast", blast_width=0.08, theta=0.02,
               coarsen_frac=0.25, weno_eps=1e-6, gamma=1.4, cfl=0.4, subcycle=1)
    run_pair(cfg, steps=10, regrid_every=4, check_each=True)


def test_shock_bubble_subcycled():
    cfg = dict(W.shock_bubble(Nx=128, Ny=64, n=16, levels=3), subcycle=1)
    run_pair(cfg, steps=10, cfl=0.5, regrid_every=4)


def test_single_level_is_the_global_step_bitwise():
    res = []
    for sub in (0, 1):
        cfg = dict(W.vortex(N=128, n=32), subcycle=sub)
        g = amr.Mesh(cfg)
        g.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
        for _ in range(3):
            g.step(cfl=0.5)
        res.append(g.get_state(as_dict=False))
    assert np.array_equal(res[0], res[1])


def test_conservation_periodic_three_levels():
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(64, 64), n=16, levels=3, bc=("periodic",) * 4,
               scheme="weno5", characteristic=1, div_order=4, ic="blast", blast_width=0.08, theta=0.02,
               coarsen_frac=0.25, weno_eps=1e-6, gamma=1.4, subcycle=1)
    g = amr.Mesh(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    g.set_state(fn)
    for _ in range(2):
        g.regrid()
        g.set_state(fn)
    assert len({k[0] for k in g.leaves()}) == 3
    t0, _ = g.diagnostics()
    st = g.get_state()
    leaves = set(g.leaves())
    scale = sum(np.abs(U).sum(axis=(1, 2)) * (1.0 / (64 << l)) ** 2 for (l, P, Q), U in st.items() if (l, P, Q) in leaves)
    for s in range(1, 9):
        g.step(cfl=0.4)
        if s % 4 == 0:
            g.regrid()
    t1, _ = g.diagnostics()
    assert np.all(np.abs(t1 - t0) <= 1e-12 * scale), (t1 - t0) / scale
