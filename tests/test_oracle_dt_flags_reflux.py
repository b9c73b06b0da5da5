"""Pins of the oracle's wave-speed / dt (O13, S6), of the flag ambiguity band (A32) and of the reflux
placement (O12), each against something other than the oracle itself:

- O13 / SPEC compute_dt: rest gas -> dt = cfl h / (2 sqrt 1.4) (printed example), on a mesh with
  dx != dy the closed form sqrt(1.4) (1/dx + 1/dy); refining every patch halves dt (printed example); the
  implosion IC (Eq. 13) on 1024^2 against the analytic maximum sound speed; random moving states on a 3-level
  mesh against a brute-force numpy maximum over the primitives (each leaf with its own level spacing); a NaN
  cell makes Lambda NaN wherever it sits.
- S6 (subcycling): the per-leaf value is divided by 2^l, so refining every patch leaves it
  unchanged; brute force on the 3-level mesh.
- A32: a density ramp whose exact indicator (rational arithmetic on the input doubles) puts one cell at
  theta (1 +- 5e-10) or theta/4 (1 +- 5e-10) must raise the ambiguity bit; at +-5e-9 it must not, and the
  refine / coarsen decision follows the strict comparisons of O6 / A20.
- O12: one stage on a 2-level strip, with and without the correction: the change is confined to the coarse
  cells adjacent to the coarse/fine faces and equals dt sigma (F_coarse - mean of the two fine faces) / h,
  computed here from the pinned composite ghost tiles and the pinned face flux; omitting it breaks
  conservation (the control the conservation pin needs).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle as orc
import workloads as W

SQ14 = math.sqrt(1.4)


def _uniform_cfg(base=(16, 16), hi=(1.0, 1.0), levels=2, n=8, state=(1.0, 0.0, 0.0, 1.0), **kw):
    c = dict(lo=(0.0, 0.0), hi=hi, base=base, n=n, levels=levels, bc=("periodic",) * 4, scheme="weno5",
             characteristic=1, div_order=4, ic="uniform", uniform_state=state)
    c.update(kw)
    return c


def _fill(o, cfg):
    o.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))


# ----------------------------------------------------------------------------- O13 / S6
def test_dt_rest_gas_printed_example():
    """rest gas rho = p = 1, gamma 1.4, dx = dy = h -> dt = cfl h / (2 sqrt 1.4)."""
    cfg = _uniform_cfg()
    o = orc.Oracle(cfg)
    _fill(o, cfg)
    h = 1.0 / 16
    cfl = 0.45
    dt = cfl / o.lam()
    assert abs(dt - cfl * h / (2.0 * SQ14)) <= 1e-15 * dt
    assert o.step(cfl=cfl) == pytest.approx(cfl * h / (2.0 * SQ14), rel=1e-15)


def test_lambda_is_the_sum_of_the_axis_radii_with_unequal_spacing():
    """O13: (|u|+c)/dx + (|v|+c)/dy -- with dx = 1/16, dy = 1/8 and u = 0.3, v = -0.7 a max of the two radii,
    a swapped spacing or a signed velocity would all give another value."""
    u, v = 0.3, -0.7
    cfg = _uniform_cfg(hi=(1.0, 2.0), state=(1.0, u, v, 1.0))
    o = orc.Oracle(cfg)
    _fill(o, cfg)
    dx, dy = 1.0 / 16, 2.0 / 16
    expect = (abs(u) + SQ14) / dx + (abs(v) + SQ14) / dy
    assert o.lam() == pytest.approx(expect, rel=1e-14)


def test_refining_every_patch_halves_dt_and_keeps_the_subcycled_lambda():
    """refining every patch once (same state) halves dt.  S6: the level-normalised Lambda of the
    subcycled step is unchanged (each level then runs at the same CFL)."""
    cfg = _uniform_cfg(levels=3, state=(1.0, 0.2, 0.1, 1.0))
    o = orc.Oracle(cfg)
    _fill(o, cfg)
    lam0, sub0 = o.lam(), o.lam_subcycled()
    assert lam0 == sub0
    o.regrid_with_requests([(0, P, Q) for Q in range(2) for P in range(2)])
    _fill(o, cfg)
    assert all(k[0] == 1 for k in o.leaves())
    assert o.lam() == 2.0 * lam0          # power-of-two spacing: exact
    assert o.lam_subcycled() == sub0
    o.regrid_with_requests([k for k in o.leaves()])
    _fill(o, cfg)
    assert all(k[0] == 2 for k in o.leaves())
    assert o.lam() == 4.0 * lam0 and o.lam_subcycled() == sub0


def test_dt_implosion_ic_brute_force():
    """Eq. (13) implosion IC on 1024^2 of (-0.3, 0.3)^2, cfl 0.45: the fastest cells are the
    low-density interior (rho, p) = (0.125, 0.14) at rest, so Lambda = 2 sqrt(1.4 * 0.14 / 0.125) / h."""
    cfg = W.implosion(N=1024, n=32, scheme="central4")
    o = orc.Oracle(cfg)
    _fill(o, cfg)
    h = 0.6 / 1024
    expect = 2.0 * math.sqrt(1.4 * 0.14 / 0.125) / h
    assert o.lam() == pytest.approx(expect, rel=1e-14)
    assert o.step(cfl=0.45) == pytest.approx(0.45 / expect, rel=1e-14)


def _three_level_mesh():
    cfg = _uniform_cfg(base=(32, 16), hi=(2.0, 1.0), levels=3)
    o = orc.Oracle(cfg)
    o.regrid_with_requests([(0, 1, 0), (0, 2, 1)])
    o.regrid_with_requests([(1, 3, 1)])
    assert {k[0] for k in o.leaves()} == {0, 1, 2}
    return cfg, o


@pytest.mark.parametrize("fast_level", [0, 1, 2])
def test_lambda_brute_force_on_three_levels(fast_level):
    """Random primitive states (u, v of both signs) on a 3-level mesh, the fastest gas placed on one level: the
    oracle's Lambda and its S6 variant equal a numpy maximum over the primitives that were set, each leaf with
    its own dx_l, dy_l (a level-0 spacing everywhere or a missing 2^-l would move the maximum by 2x or 4x)."""
    cfg, o = _three_level_mesh()
    n = cfg["n"]
    rng = np.random.default_rng(11 + fast_level)
    lam_bf, sub_bf = 0.0, 0.0
    for (l, P, Q, leaf) in o.tree():
        rho = rng.uniform(0.5, 2.0, (n, n))
        p = rng.uniform(0.5, 2.0, (n, n))
        boost = 6.0 if l == fast_level else 1.0
        u = boost * rng.uniform(-1, 1, (n, n))
        v = boost * rng.uniform(-1, 1, (n, n))
        o.set_patch((l, P, Q), W.to_conserved(rho, u, v, p))
        if leaf:
            dx = 2.0 / (32 << l)
            dy = 1.0 / (16 << l)
            c = np.sqrt(1.4 * p / rho)
            s = (np.abs(u) + c) / dx + (np.abs(v) + c) / dy
            lam_bf = max(lam_bf, s.max())
            sub_bf = max(sub_bf, s.max() / (1 << l))
    assert o.lam() == pytest.approx(lam_bf, rel=1e-13)
    assert o.lam_subcycled() == pytest.approx(sub_bf, rel=1e-13)


@pytest.mark.parametrize("where", ["first", "middle", "last"])
def test_lambda_nan_is_sticky(where):
    """A non-physical cell (p < 0: c = sqrt(negative) = NaN) makes Lambda NaN wherever the cell sits in the
    leaf order (a later finite cell must not replace it), and a CFL step then fails without committing."""
    cfg, o = _three_level_mesh()
    _fill(o, cfg)
    leaves = o.leaves()
    key = {"first": leaves[0], "middle": leaves[len(leaves) // 2], "last": leaves[-1]}[where]
    U = o.get_patch(key)
    U[3, 2, 3] = -1.0            # E < 0 at rest -> p < 0
    o.set_patch(key, U)
    assert math.isnan(o.lam()) and math.isnan(o.lam_subcycled())
    before = o.get_state()
    with pytest.raises(orc.OracleError) as ei:
        o.step(cfl=0.5)
    assert ei.value.code == 3
    after = o.get_state()
    assert all(np.array_equal(before[k], after[k], equal_nan=True) for k in before)


# ----------------------------------------------------------------------------- A32 ambiguity band
def ramp_case(kind, delta):
    """Density ramp rho_i = 1 + s i along x (u = v = 0, p = 1), constant in y (periodic y, transmissive x), so
    interior cells have eta_i = s / (1 + s i) exactly in real arithmetic.
    kind 'refine':  one level-0 row of 4 leaves; s chosen so that eta_1 = theta (1 + delta) (cell 1 is the
                    maximum: cell 0 sees the zero-gradient ghost, eta_0 = s / 2).
    kind 'coarsen': every root refined (levels 2); s chosen so that the first fine cell of root 1, i = 16,
                    has eta = theta/4 (1 + delta); that cell is root 1's children's maximum.
    Returns (cfg, builder(o) that sets the state, the row of rho values)."""
    theta = 0.1
    n = 8
    if kind == "refine":
        t = theta * (1.0 + delta)
        s = t / (1.0 - t)
        ncell, lev = 32, 0
    else:
        t = 0.25 * theta * (1.0 + delta)
        s = t / (1.0 - 16.0 * t)
        ncell, lev = 64, 1
    rho = 1.0 + s * np.arange(ncell, dtype=np.float64)
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 0.25), base=(32, 8), n=n, levels=2,
               bc=("transmissive", "transmissive", "periodic", "periodic"), scheme="weno5", characteristic=1,
               div_order=4, theta=theta, coarsen_frac=0.25, ic="uniform", uniform_state=(1.0, 0.0, 0.0, 1.0))

    def state(l, P, Q):
        r = 1.0 + s * np.arange(P * n, P * n + n, dtype=np.float64)   # the same doubles as `rho`
        if l != lev:                   # covered level-0 patches: overwritten by the restriction anyway
            r = np.ones(n)
        R = np.broadcast_to(r[None, :], (n, n))
        z = np.zeros((n, n))
        return W.to_conserved(R, z, z, z + 1.0)

    return cfg, state, rho, lev


def exact_eta(rho, dx):
    """eta_i = dx |(rho_{i+1} - rho_{i-1}) / (2 dx)| / rho_i over the row in rational arithmetic on the given
    doubles (zero-gradient ghosts at both ends; the y-gradient is exactly zero)."""
    r = [Fraction(float(x)) for x in rho]
    N = len(r)
    d = Fraction(dx)
    out = []
    for i in range(N):
        a = r[i + 1] if i + 1 < N else r[N - 1]
        b = r[i - 1] if i >= 1 else r[0]
        out.append(abs(d * ((a - b) / (2 * d))) / r[i])
    return out


def expected_flags(kind, rho, lev, theta=0.1):
    """Per leaf / parent the O6 / A20 / A32 decisions from the exact eta, with the margins asserted so that
    floating-point evaluation (relative error ~1e-15) cannot flip them."""
    dx = 1.0 / (32 << lev)
    eta = exact_eta(rho, dx)
    th, tc = Fraction(theta), Fraction(theta) / 4
    for e in eta:   # every cell is either far outside the band or well inside it
        for T in (th, tc):
            r = abs(e - T) / T
            assert r < Fraction(9, 10**10) or r > Fraction(11, 10**10) or r == 0
            assert abs(r - Fraction(1, 10**9)) > Fraction(1, 10**11)
    amb = [any(abs(e - T) <= Fraction(1, 10**9) * T for T in (th, tc)) for e in eta]
    if kind == "refine":
        return {P: (max(eta[8 * P:8 * P + 8]) > th, any(amb[8 * P:8 * P + 8])) for P in range(4)}
    return {P: (max(eta[16 * P:16 * P + 16]) < tc, any(amb[16 * P:16 * P + 16])) for P in range(4)}


def build_ramp(mesh, kind, state):
    mesh.set_state(state)
    if kind == "coarsen":
        mesh.regrid_with_requests([(0, P, 0) for P in range(4)])
        mesh.set_state(state)


@pytest.mark.parametrize("kind", ["refine", "coarsen"])
@pytest.mark.parametrize("delta", [5e-10, -5e-10, 5e-9, -5e-9])
def test_ambiguity_band(kind, delta):
    cfg, state, rho, lev = ramp_case(kind, delta)
    exp = expected_flags(kind, rho, lev)
    # the constructed cell really sits where the case says
    inside = abs(delta) < 1e-9
    assert exp[0 if kind == "refine" else 1][1] == inside
    o = orc.Oracle(cfg)
    build_ramp(o, kind, state)
    fl = o.flags()
    for P in range(4):
        me, rf, cf, am = fl[(0, P, 0)]
        dec, amb = exp[P]
        assert am == amb, (P, me, am, amb)
        assert (rf if kind == "refine" else cf) == dec, (P, me, dec)
    # the decision at the constructed cell follows the sign of delta (strict comparisons)
    P0 = 0 if kind == "refine" else 1
    assert exp[P0][0] == (delta > 0 if kind == "refine" else delta < 0)


# ----------------------------------------------------------------------------- O12 reflux placement
def _fhat_line(o, key, axis, line):
    """F-hat (Eq. 9 flux form, O10) at the faces m = 0..n of one row (axis 0) or column (axis 1) of leaf `key`,
    from its composite ghost tile (O7, pinned in test_oracle_scheme) and the pinned unit face flux."""
    n, g = o.n, 4
    T = o.ghost_tile(key, g)       # [4][n+2g][n+2g], index [k][j+g][i+g]
    f = {}
    for m in range(-1, n + 2):
        if axis == 0:
            cells = np.array([T[:, line + g, m - 3 + s + g] for s in range(6)])
        else:
            cells = np.array([T[[0, 2, 1, 3], m - 3 + s + g, line + g] for s in range(6)])
        fm = orc.face_flux_x(o.cfg, cells)
        f[m] = fm if axis == 0 else fm[[0, 2, 1, 3]]
    return {m: 13.0 / 12.0 * f[m] - 1.0 / 24.0 * (f[m - 1] + f[m + 1]) for m in range(0, n + 1)}


@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("scheme", ["weno5", "central4"])
def test_reflux_placement_single_stage(axis, scheme):
    """O12 on a 2-level periodic strip (one refined root, dx0 != dy0): one stage with the correction minus the
    same stage without it is non-zero only in the coarse cells next to the two C/F faces, where it equals
    b_1 dt sigma (F_c - (F_f1 + F_f2)/2) / h_axis; sigma = +1 on the coarse cell's high side."""
    n = 8
    if axis == 0:
        base, hi, refined, ic = (32, 8), (1.0, 0.5), (0, 1, 0), dict(u0=0.8, v0=0.0)
    else:
        base, hi, refined, ic = (8, 32), (0.5, 1.0), (0, 0, 1), dict(u0=0.0, v0=0.8)
    cfg = dict(lo=(0.0, 0.0), hi=hi, base=base, n=n, levels=2, bc=("periodic",) * 4, scheme=scheme,
               characteristic=1, div_order=4, ic="uniform", **ic)

    def state(l, P, Q):
        X, Y = W.cell_centres(cfg, l, P, Q)
        s = X if axis == 0 else Y
        rho = 1.0 + 0.3 * np.sin(2 * math.pi * s)
        z = np.zeros_like(X)
        return W.to_conserved(rho, z + ic["u0"], z + ic["v0"], z + 1.0)

    runs = {}
    for on in (1, 0):
        o = orc.Oracle(dict(cfg, oracle_reflux=on))
        o.set_state(state)
        o.regrid_with_requests([refined])
        o.set_state(state)
        dt = 0.5 / o.lam()
        o.stage1(dt)
        runs[on] = (o.get_state(), dt)
    Son, dt = runs[1]
    Soff = runs[0][0]
    o = orc.Oracle(cfg)              # the stage input, for the face fluxes
    o.set_state(state)
    o.regrid_with_requests([refined])
    o.set_state(state)
    h = (hi[axis] - 0.0) / (base[axis])
    expect = {k: np.zeros_like(v) for k, v in Son.items()}
    # the coarse neighbours of the refined root: low neighbour (its high side faces the fine patches) and high
    lo_key = (0, 0, 0)
    hi_key = (0, 2, 0) if axis == 0 else (0, 0, 2)
    for key, sigma in ((lo_key, +1.0), (hi_key, -1.0)):
        for t in range(n):
            Fc = _fhat_line(o, key, axis, t)[n if sigma > 0 else 0]
            # global coarse cell and the two fine cells across the face
            Ic = key[1] * n + (n - 1 if (axis == 0 and sigma > 0) else 0 if axis == 0 else t)
            Jc = key[2] * n + (n - 1 if (axis == 1 and sigma > 0) else 0 if axis == 1 else t)
            Ff = []
            for b in range(2):
                if axis == 0:
                    fI = 2 * Ic + 2 if sigma > 0 else 2 * Ic - 1
                    fJ = 2 * Jc + b
                    fkey = (1, fI // n, fJ // n)
                    line, m = fJ % n, 0 if sigma > 0 else n
                else:
                    fI = 2 * Ic + b
                    fJ = 2 * Jc + 2 if sigma > 0 else 2 * Jc - 1
                    fkey = (1, fI // n, fJ // n)
                    line, m = fI % n, 0 if sigma > 0 else n
                Ff.append(_fhat_line(o, fkey, axis, line)[m])
            corr = dt * sigma * (Fc - 0.5 * (Ff[0] + Ff[1])) / h
            ci, cj = Ic - key[1] * n, Jc - key[2] * n
            expect[key][:, cj, ci] = corr
    big = 0.0
    for k in Son:
        d = Son[k] - Soff[k]
        scale = np.abs(Son[k]).max()
        assert np.all(np.abs(d - expect[k]) <= 4e-16 * scale), (k, np.abs(d - expect[k]).max())
        big = max(big, np.abs(expect[k]).max())
    assert big > 1e-9      # the correction is real, not rounding (so the placement is actually tested)


def test_no_reflux_control_breaks_conservation():
    """Control for the conservation pin (test_oracle_scheme): the same 2-level strip and smooth moving wave without
    the O12 correction changes the leaf totals by far more than rounding, with it they telescope (<= 1e-13)."""
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 0.25), base=(32, 8), n=8, levels=2, bc=("periodic",) * 4,
               scheme="weno5", characteristic=1, div_order=4, ic="smooth", amp=0.3, u0=0.8, v0=0.0)
    drift = {}
    for on in (1, 0):
        o = orc.Oracle(dict(cfg, oracle_reflux=on))
        _fill(o, cfg)
        o.regrid_with_requests([(0, 1, 0)])
        _fill(o, cfg)
        t0 = o.totals()
        for _ in range(5):
            o.step(cfl=0.5)
        drift[on] = abs(o.totals()[0] - t0[0]) / abs(t0[0])
    assert drift[1] < 1e-13
    assert drift[0] > 1e-9, drift
