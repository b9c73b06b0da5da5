"""Pins of the oracle's Berger-Colella time subcycling (NEXT #4; readings S1-S6 in oracle/oracle.cpp and
DESIGN.md s3b): reduction to the global-dt scheme where the two must coincide, free stream, conservation with the
accumulated flux registers across coarse/fine interfaces, and accuracy against the exact Riemann solution."""
import numpy as np
import pytest

import oracle as orc
import workloads as W
from tests import exact_riemann as ER
from tests.test_oracle_scheme import _totals_scale, rel_change, run_init


def _state(o):
    return {k: v.copy() for k, v in o.get_state().items()}


@pytest.mark.parametrize("scheme", ["central4", "weno5"])
def test_single_level_equals_global_step(scheme):
    """S1 with one level: one subcycled step is the O11 step, bit for bit."""
    cfg = W.vortex(N=64, n=16, scheme=scheme)
    a, b = orc.Oracle(cfg), orc.Oracle(cfg)
    for o in (a, b):
        o.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    for _ in range(3):
        d1 = a.step(cfl=0.5)
        d2 = b.step(cfl=0.5, subcycle=True)
        assert d1 == d2
    sa, sb = a.get_state(), b.get_state()
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k


@pytest.mark.parametrize("scheme", ["central4", "weno5"])
def test_fully_refined_equals_two_fine_steps(scheme):
    """S1/S2: with every root refined, the leaves see no coarse/fine face; one subcycled step of dt must equal two
    global steps of dt/2 on the leaves, bit for bit, and the covered level is their restriction."""
    cfg = dict(W.vortex(N=32, n=8, scheme=scheme), levels=2)
    a, b = orc.Oracle(cfg), orc.Oracle(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    roots = [(0, P, Q) for P in range(4) for Q in range(4)]
    for o in (a, b):
        o.set_state(fn)
        o.regrid_with_requests(roots, [])
        o.set_state(fn)
    dt = 0.4 / a.lam()
    a.step(dt=dt, subcycle=True)
    for _ in range(2):
        b.step(dt=0.5 * dt)
    sa, sb = a.get_state(), b.get_state()
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k


@pytest.mark.parametrize("bcname", ["periodic", "mixed"])
def test_free_stream_preserved(bcname):
    """A uniform state on a 3-level mesh stays uniform: time interpolation of equal states is exact, every face
    flux is equal; the register sums over 3 (coarse) and 6 (fine) weighted terms can differ in the last bit, so
    the bound is 4 ulp rather than bitwise (the global-dt scheme's free-stream test is bitwise)."""
    bc = ("periodic",) * 4 if bcname == "periodic" else ("transmissive", "transmissive", "reflective", "reflective")
    state = (1.3, 0.4, -0.25, 0.9) if bcname == "periodic" else (1.3, 0.4, 0.0, 0.9)
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(32, 32), n=8, levels=3, bc=bc, scheme="weno5",
               characteristic=1, div_order=4, ic="uniform", uniform_state=state)
    o = orc.Oracle(cfg)
    o.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    o.regrid_with_requests([(0, 1, 1), (0, 2, 1), (0, 0, 3)])
    o.regrid_with_requests([(1, 3, 3), (1, 2, 2)])
    o.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    before = _state(o)
    assert len({k[0] for k in before}) == 3
    for _ in range(3):
        o.step(cfl=0.5, subcycle=True)
    after = o.get_state()
    for k in before:
        assert np.all(np.abs(after[k] - before[k]) <= 4 * np.spacing(np.abs(before[k]))), k


@pytest.mark.parametrize("scheme", ["central4", "weno5"])
def test_conservation_periodic_amr(scheme):
    """S3/S4: the accumulated registers make the subcycled composite update conservative to 1e-12 across
    coarse/fine interfaces of a 3-level periodic mesh, with regrids between steps."""
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(32, 32), n=8, levels=3, bc=("periodic",) * 4,
               scheme=scheme, characteristic=1, div_order=4, ic="blast", blast_width=0.08,
               theta=0.02, coarsen_frac=0.25, weno_eps=1e-6, gamma=1.4)
    o = orc.Oracle(cfg)
    run_init(o, cfg)
    assert len({l for (l, _, _, lf) in o.tree() if lf}) == 3
    t0, sc = o.totals(), _totals_scale(o)
    for s in range(1, 7):
        o.step(cfl=0.4, subcycle=True)
        if s % 3 == 0:
            o.regrid()
    assert np.all(rel_change(o.totals(), t0, sc) < 1e-12), rel_change(o.totals(), t0, sc)


def test_subcycled_differs_from_global_dt_on_amr():
    """Control for the pins above: on a 2-level mesh with a moving front the subcycled integration is genuinely
    a different time discretisation from the global-dt one (so the conservation pin tests its registers)."""
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(32, 32), n=8, levels=2, bc=("periodic",) * 4,
               scheme="weno5", characteristic=1, div_order=4, ic="blast", blast_width=0.08,
               theta=0.02, coarsen_frac=0.25, weno_eps=1e-6, gamma=1.4)
    a, b = orc.Oracle(cfg), orc.Oracle(cfg)
    for o in (a, b):
        run_init(o, cfg)
    dt = 0.4 / a.lam()
    a.step(dt=dt, subcycle=True)
    b.step(dt=dt)
    sa, sb = a.get_state(), b.get_state()
    gap = max(np.abs(sa[k] - sb[k]).max() for k in sa)
    assert gap > 1e-8    # the two time integrations genuinely differ


def test_sod_subcycled_against_exact_riemann():
    """S1-S6 accuracy: BJ configs[0] (A21/A23 strip, 2 levels) to t = 0.2 with subcycling; L1(rho) vs O16."""
    cfg = dict(W.sod(), base=(208, 8), n=8, hi=(1.04, 0.04))
    o = orc.Oracle(cfg)
    run_init(o, cfg)
    t, step = 0.0, 0
    while t < 0.2 - 1e-15:
        lam = o.lam()
        d = min(0.5 * 2.0 / lam, 0.2 - t)          # level-0 step: every level at CFL <= 0.5 (S6, 2 levels)
        o.step(dt=d, subcycle=True)
        t += d
        step += 1
        if step % 2 == 0:
            o.regrid()
    err = 0.0
    for (l, P, Q, lf) in o.tree():
        if lf and Q == 0:
            U = o.get_patch((l, P, Q))
            X, Y = W.cell_centres(cfg, l, P, Q)
            m = X[0] < 1.0
            ex, _, _ = ER.sample(1.0, 0.0, 1.0, 0.125, 0.0, 0.1, (X[0][m] - 0.5) / 0.2)
            err += np.sum(np.abs(U[0][0][m] - ex)) * 0.005 / (1 << l)
    assert err < 0.012, err
