"""Pins of the oracle's patch tree (Alg. 1 / Alg. 2, rules R1 / R2) and refinement flags (O6).

The validity checker and the minimal-closure enumeration below are written independently of the oracle
(set fix-points in Python), so they pin Alg. 1 / Alg. 2 rather than restate them.
"""
import itertools
import random

import numpy as np
import pytest

import oracle as orc
import workloads as W

MOORE = [(0, 1), (1, 0), (0, -1), (-1, 0), (1, 1), (1, -1), (-1, -1), (-1, 1)]


def small_cfg(nr=4, levels=4, periodic=True, n=8, **kw):
    bc = ("periodic",) * 4 if periodic else ("transmissive",) * 4
    c = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(nr * n, nr * n), n=n, levels=levels, bc=bc,
             scheme="central4", ic="uniform", gamma=1.4, theta=0.1, coarsen_frac=0.25)
    c.update(kw)
    return c


def uniform_oracle(cfg):
    o = orc.Oracle(cfg)
    o.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    return o


def keyset(o):
    return {(l, P, Q) for (l, P, Q, _) in o.tree()}


def _wrap(cfg, l, P, Q):
    npx = (cfg["base"][0] // cfg["n"]) << l
    npy = (cfg["base"][1] // cfg["n"]) << l
    per = cfg["bc"][0] == "periodic"
    if not per and not (0 <= P < npx and 0 <= Q < npy):
        return None
    return (l, P % npx, Q % npy)


def valid(cfg, keys):
    """Independent statement of R1, R2 and all-or-none children."""
    npx, npy = cfg["base"][0] // cfg["n"], cfg["base"][1] // cfg["n"]
    if not all((0, P, Q) in keys for P in range(npx) for Q in range(npy)):
        return False
    for (l, P, Q) in keys:
        kids = [(l + 1, 2 * P + a, 2 * Q + b) in keys for a in (0, 1) for b in (0, 1)]
        if any(kids) and not all(kids):
            return False
        if l > 0 and (l - 1, P // 2, Q // 2) not in keys:
            return False
        if all(kids):
            for dx, dy in MOORE:
                k = _wrap(cfg, l, P + dx, Q + dy)
                if k is not None and k not in keys:
                    return False
    return True


def has_children(keys, k):
    return (k[0] + 1, 2 * k[1], 2 * k[2]) in keys


def refine_via(o, keys):
    return o.regrid_with_requests(refine_keys=keys)


def test_trivial_counts():
    """refining one level-0 patch of a 4x4 periodic scaffold adds exactly 4 patches, 19 leaves."""
    cfg = small_cfg()
    o = uniform_oracle(cfg)
    assert len(o.tree()) == 16
    refine_via(o, [(0, 1, 2)])
    assert len(o.tree()) == 20 and len(o.leaves()) == 19
    o.validate()


def test_fig5_recursive_refinement():
    """P:L257 / Fig. 5 (A37): refining a level-1 leaf whose level-1 Moore neighbour across its parent's edge
    is missing must first refine the adjacent root (Alg. 1 line 6-7)."""
    cfg = small_cfg(periodic=False)
    o = uniform_oracle(cfg)
    refine_via(o, [(0, 1, 1)])
    # child (1, 3, 3) is the NE child of root (1,1): its E/NE/N neighbours live in roots (2,1),(2,2),(1,2)
    refine_via(o, [(1, 3, 3)])
    ks = keyset(o)
    assert (2, 6, 6) in ks
    for root in [(0, 2, 1), (0, 2, 2), (0, 1, 2)]:
        assert has_children(ks, root), root
    assert not has_children(ks, (0, 0, 0))
    assert valid(cfg, ks)


def _closure(cfg, keys, p):
    """Smallest valid superset of `keys` in which p has children: fix-point of 'add the 4 children of
    the parent of any missing Moore position of a patch that has children'."""
    ks = set(keys) | {(p[0] + 1, 2 * p[1] + a, 2 * p[2] + b) for a in (0, 1) for b in (0, 1)}
    changed = True
    while changed:
        changed = False
        for (l, P, Q) in list(ks):
            if not has_children(ks, (l, P, Q)):
                continue
            for dx, dy in MOORE:
                k = _wrap(cfg, l, P + dx, Q + dy)
                if k is None or k in ks:
                    continue
                par = (l - 1, k[1] // 2, k[2] // 2)
                ks |= {(l, 2 * par[1] + a, 2 * par[2] + b) for a in (0, 1) for b in (0, 1)}
                changed = True
    return ks


@pytest.mark.parametrize("nr,periodic", [(2, True), (3, True), (3, False)])
def test_alg1_equals_minimal_closure_bruteforce(nr, periodic):
    cfg = small_cfg(nr=nr, levels=3, periodic=periodic)
    rng = random.Random(nr * 10 + periodic)
    for trial in range(40):
        o = uniform_oracle(cfg)
        for _ in range(rng.randint(1, 4)):
            leaves = [k for k in o.leaves() if k[0] < cfg["levels"] - 1]
            p = rng.choice(leaves)
            before = keyset(o)
            refine_via(o, [p])
            after = keyset(o)
            assert after == _closure(cfg, before, p)
            assert valid(cfg, after)


def test_fuzz_validity_refine_and_coarsen():
    """S:L603 (reduced count): random request sequences on 4x4 periodic roots, max level 4: every mesh valid."""
    cfg = small_cfg(nr=4, levels=4)
    rng = random.Random(7)
    for seq in range(60):
        o = uniform_oracle(cfg)
        for it in range(rng.randint(2, 6)):
            tr = o.tree()
            leaves = [(l, P, Q) for (l, P, Q, lf) in tr if lf and l < 3]
            parents = [(l, P, Q) for (l, P, Q, lf) in tr if not lf]
            ref = rng.sample(leaves, min(len(leaves), rng.randint(0, 3)))
            crs = rng.sample(parents, min(len(parents), rng.randint(0, 3)))
            o.regrid_with_requests(ref, crs)
            assert valid(cfg, keyset(o))


def test_refine_then_coarsen_round_trip():
    cfg = small_cfg()
    o = uniform_oracle(cfg)
    before = keyset(o)
    refine_via(o, [(0, 2, 2)])
    o.regrid_with_requests(coarsen_keys=[(0, 2, 2)])
    assert keyset(o) == before


def test_coarsen_rules_r2_exact_vs_alg2_literal():
    """A16: two adjacent refined roots block each other under the literal Alg. 2 and also the
    level-0 guard makes level-1 parents permanent; the R2-exact prose rule deletes them."""
    for rule, expect_deleted in (("alg2_literal", False), ("r2_exact", True)):
        cfg = small_cfg(coarsen_rule=rule)
        o = uniform_oracle(cfg)
        refine_via(o, [(0, 1, 1), (0, 2, 1)])
        o.regrid_with_requests(coarsen_keys=[(0, 1, 1)])
        ks = keyset(o)
        assert has_children(ks, (0, 1, 1)) != expect_deleted
        assert valid(cfg, ks)
    # R2-exact keeps a coarsening that would break support of a finer patch
    cfg = small_cfg(nr=4, levels=3, periodic=False)
    o = uniform_oracle(cfg)
    refine_via(o, [(0, 1, 1)])
    refine_via(o, [(1, 3, 3)])          # forces roots (2,1),(2,2),(1,2) to refine
    o.regrid_with_requests(coarsen_keys=[(0, 2, 2)])
    assert has_children(keyset(o), (0, 2, 2))   # its children support (1,3,3)'s children


def test_coarsening_order_independent_within_level():
    """O5: within one level, the accepted set equals 'each request tested against the pre-pass mesh'."""
    cfg = small_cfg(nr=4, levels=3)
    rng = random.Random(3)
    for trial in range(30):
        o = uniform_oracle(cfg)
        leaves = [k for k in o.leaves()]
        o.regrid_with_requests(rng.sample(leaves, 5))
        ks = keyset(o)
        lvl0_parents = [k for k in ks if k[0] == 0 and has_children(ks, k)
                        and not any(has_children(ks, (1, 2 * k[1] + a, 2 * k[2] + b)) for a in (0, 1) for b in (0, 1))]
        req = rng.sample(lvl0_parents, min(3, len(lvl0_parents)))
        # independent evaluation: allowed iff no level-1 non-sibling patch with children touches its children
        expect = set(ks)
        for p in req:
            ok = True
            for a, b in itertools.product((0, 1), repeat=2):
                ch = (1, 2 * p[1] + a, 2 * p[2] + b)
                for dx, dy in MOORE:
                    q = _wrap(cfg, 1, ch[1] + dx, ch[2] + dy)
                    if q and (q[1] // 2, q[2] // 2) != (p[1], p[2]) and has_children(ks, q):
                        ok = False
            if ok:
                expect -= {(1, 2 * p[1] + a, 2 * p[2] + b) for a in (0, 1) for b in (0, 1)}
        o.regrid_with_requests(coarsen_keys=req)
        assert keyset(o) == expect


# ----------------------------------------------------------------------------- flags (O6)
def test_flags_uniform_none():
    cfg = small_cfg(levels=2)
    o = uniform_oracle(cfg)
    fl = o.flags()
    assert not any(v[1] for v in fl.values())
    assert all(v[0] == 0.0 for k, v in fl.items())


def test_flags_linear_ramp_closed_form():
    """rho = 1 + a x, uniform p, u: eta = dx * a / rho exactly (central difference exact on linears)."""
    a = 0.9
    cfg = dict(small_cfg(nr=4, levels=2, periodic=False), ic="smooth")
    o = orc.Oracle(cfg)

    def fn(l, P, Q):
        X, Y = W.cell_centres(cfg, l, P, Q)
        return W.to_conserved(1.0 + a * X, 0 * X + 0.1, 0 * X, 0 * X + 1.0)

    o.set_state(fn)
    fl = o.flags()
    dx = 1.0 / 32
    for (l, P, Q), (me, rf, cf, am) in fl.items():
        X, Y = W.cell_centres(cfg, l, P, Q)
        # interior columns only see exact central differences; boundary clamp halves the difference
        eta = dx * a / (1.0 + a * X)
        inner = eta[:, 1:-1] if P in (0, 3) else eta
        assert me >= inner.max() * (1 - 1e-12)
        assert me <= eta.max() * (1 + 1e-12)
        assert rf == (me > 0.1)


def test_flags_threshold_and_coarsen_requests():
    cfg = dict(small_cfg(nr=4, levels=3, periodic=True), theta=0.1, coarsen_frac=0.25)
    o = orc.Oracle(cfg)

    def fn(l, P, Q):
        X, Y = W.cell_centres(cfg, l, P, Q)
        return W.to_conserved(1.0 + 2.0 * np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / 0.005), 0 * X, 0 * X, 1 + 0 * X)

    o.set_state(fn)
    fl = o.flags()
    ref = [k for k, v in fl.items() if v[1]]
    assert ref and all(k[0] == 0 for k in ref)
    o.regrid()
    o.set_state(fn)
    o.regrid()
    o.set_state(fn)
    fl = o.flags()
    for (l, P, Q), (me, rf, cf, am) in fl.items():
        if cf:
            assert me < 0.025


def test_flags_mirror_symmetric():
    cfg = dict(small_cfg(nr=4, levels=2, periodic=False))
    o = orc.Oracle(cfg)

    def fn(l, P, Q):
        X, Y = W.cell_centres(cfg, l, P, Q)
        return W.to_conserved(1.0 + 0.4 * np.tanh((np.abs(X - 0.5) - 0.2) / 0.02), 0 * X, 0 * X, 1 + 0 * X)

    o.set_state(fn)
    fl = o.flags()
    for (l, P, Q), v in fl.items():
        m = fl[(l, 3 - P, Q)]
        assert v[1] == m[1] and abs(v[0] - m[0]) <= 1e-12 * max(1e-300, abs(v[0]))
