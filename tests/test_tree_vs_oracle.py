"""The library's host patch tree (include/amr_debug.h, CPU only) against the oracle's independent tree under random
mixed refine / coarsen requests -- heavy on coarsening, so that the R2-exact coarsening rule (A16; PatchTree::
coarsen_allowed, which inspects the 12 level-(l+1) cells around a sibling block through the parent's Moore
neighbours) is exercised both ways -- on periodic and walled domains, 4 levels: the active patch sets agree after
every regrid."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
from tests.test_multirank_host import Plan


def _cfg(bc):
    return dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(48, 32), n=8, levels=4, bc=bc, scheme="weno5", ic="uniform")


@pytest.mark.parametrize("bc", [("periodic",) * 4, ("transmissive", "transmissive", "reflective", "reflective")])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tree_equals_oracle_under_mixed_requests(bc, seed):
    orc.build()
    cfg = _cfg(bc)
    rng = np.random.default_rng(seed)
    o = orc.Oracle(cfg)
    p = Plan(cfg)
    coarsened = 0
    for it in range(24):
        tr = p.tree(1)
        keys = [(d.level, d.i, d.j) for d in tr]
        assert set(keys) == {(l, P, Q) for (l, P, Q, _) in o.tree()}
        leaves = [e for e, d in enumerate(tr) if d.leaf and d.level < 3]
        parents = [e for e, d in enumerate(tr) if not d.leaf]
        nref = 0 if it >= 16 else min(len(leaves), int(rng.integers(1, 6)))
        ncrs = min(len(parents), int(rng.integers(len(parents) // 2, len(parents) + 1))) if parents else 0
        ref = [int(x) for x in rng.choice(leaves, size=nref, replace=False)] if nref else []
        crs = [int(x) for x in rng.choice(parents, size=ncrs, replace=False)] if ncrs else []
        bits = {}
        for e in ref:
            bits[e] = bits.get(e, 0) | 1
        for e in crs:
            bits[e] = bits.get(e, 0) | 2
        idx = np.array(sorted(bits), np.int32)
        b = np.array([bits[e] for e in idx], np.uint8)
        rc = p.L.amr_plan_regrid(p.h, len(idx), idx.ctypes.data_as(C.POINTER(C.c_int32)),
                                 b.ctypes.data_as(C.POINTER(C.c_uint8)))
        assert rc == 0
        _, nc = o.regrid_with_requests([keys[e] for e in ref], [keys[e] for e in crs])
        coarsened += nc
    assert set((d.level, d.i, d.j) for d in p.tree(1)) == {(l, P, Q) for (l, P, Q, _) in o.tree()}
    assert coarsened > 0
