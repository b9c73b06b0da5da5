"""The library's patch tree (host, CPU-only through include/amr_debug.h) after random refinement requests: every
Moore neighbour link of amr_plan_tree -- computed from parent/child links and the root table, without a hash --
equals a brute-force lookup of the neighbour's (level, i, j) among the active patches (periodic wrap in x, walls
in y), and the links are symmetric; parent/child links match the positions.  Exercises R2 closure too (Alg. 1
recursion creates the support the lookup relies on)."""
import ctypes as C

import numpy as np
import pytest

from tests.test_multirank_host import MOORE, Plan


def _cfg(levels):
    return dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(64, 48), n=8, levels=levels,
                bc=("periodic", "periodic", "reflective", "reflective"), scheme="weno5", ic="uniform")


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_neighbour_links_match_brute_force(seed):
    rng = np.random.default_rng(seed)
    levels = 4
    p = Plan(_cfg(levels))
    for _ in range(3):   # three rounds of random refinement requests on current leaves
        tr = p.tree(1)
        leaves = [(d.level, d.i, d.j) for d in tr if d.leaf and d.level < levels - 1]
        pick = rng.choice(len(leaves), size=max(1, len(leaves) // 6), replace=False)
        p.refine([leaves[k] for k in pick])
    tr = p.tree(1)
    order = [(d.level, d.j, d.i) for d in tr]   # canonical order (compact radix keys): (level, j, i), unique
    assert order == sorted(set(order))
    key = {(d.level, d.i, d.j): e for e, d in enumerate(tr)}
    npx = {l: (64 // 8) << l for l in range(levels)}
    npy = {l: (48 // 8) << l for l in range(levels)}
    assert len({d.level for d in tr}) == levels
    for e, d in enumerate(tr):
        for q, (dx, dy) in enumerate(MOORE):
            i, j = (d.i + dx) % npx[d.level], d.j + dy
            want = key.get((d.level, i, j), -1) if 0 <= j < npy[d.level] else -1
            assert d.nbr[q] == want, ((d.level, d.i, d.j), (dx, dy), d.nbr[q], want)
            if want >= 0:   # symmetric
                assert tr[want].nbr[MOORE.index((-dx, -dy))] == e
        if d.parent >= 0:
            par = tr[d.parent]
            assert (par.level, par.i, par.j) == (d.level - 1, d.i // 2, d.j // 2)
        for c in range(4):
            if d.child[c] >= 0:
                ch = tr[d.child[c]]
                assert (ch.level, ch.i, ch.j) == (d.level + 1, 2 * d.i + (c & 1), 2 * d.j + (c >> 1))


@pytest.mark.parametrize("rule", ["r2_exact", "alg2_literal"])
@pytest.mark.parametrize("seed", [0, 1])
def test_incremental_validation_matches_full(rule, seed):
    """The device path validates a regrid in O(changes) (PatchTree::validate_txn); amr_plan_regrid runs it beside
    the full O(active) validate() and returns AMR_E_STATE (8) if they ever disagree.  Random mixed refine /
    coarsen requests under both coarsening rules (the literal Alg. 2 rule can break R2 and must be rejected by
    both); a rejected regrid leaves the tree unchanged."""
    rng = np.random.default_rng(100 + seed)
    levels = 4
    p = Plan(dict(_cfg(levels), coarsen_rule=rule))
    L = p.L
    outcomes = {0: 0, 4: 0}
    sizes = []
    for it in range(14):
        tr = p.tree(1)
        sizes.append(len(tr))
        if it < 10:   # grow with mixed requests, then coarsen everywhere coarsening is allowed
            k = rng.integers(1, max(2, len(tr) // 3))
            idx = rng.choice(len(tr), size=k, replace=False).astype(np.int32)
            bits = rng.choice(np.array([1, 2, 2, 3], np.uint8), size=k)
        else:
            k = len(tr)
            idx = np.arange(k, dtype=np.int32)
            bits = np.full(k, 2, np.uint8)
        rc = L.amr_plan_regrid(p.h, k, idx.ctypes.data_as(C.POINTER(C.c_int32)),
                               bits.ctypes.data_as(C.POINTER(C.c_uint8)))
        assert rc in outcomes, rc
        outcomes[rc] += 1
        if rc:
            assert [(d.level, d.i, d.j) for d in p.tree(1)] == [(d.level, d.i, d.j) for d in tr]
    sizes.append(len(p.tree(1)))
    order = [(d.level, d.j, d.i) for d in p.tree(1)]
    assert order == sorted(set(order))
    assert outcomes[0] > 0
    assert min(sizes[10:]) < sizes[10] and sizes[10] > sizes[0]   # grew, then shrank
