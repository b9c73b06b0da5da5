"""amr_regrid's device-side flag compaction (flag evaluation + compaction) against the full per-patch
flags of amr_get_flags: on two meshes with identical states, amr_regrid (compact (slot, bits) list from the device)
and amr_regrid_with_flags fed the mesh's own full flags must produce the same tree and bitwise the same state,
regrid after regrid, through refinements and coarsenings."""
import numpy as np
import pytest

import paper_2508_05020_b200 as amr
import workloads as W

pytestmark = pytest.mark.gpu


def _own_requests(g):
    f = g.flags()
    return [k for k, v in f.items() if v[1]], [k for k, v in f.items() if v[2]]


@pytest.mark.parametrize("name", ["quadrant", "shock_bubble"])
def test_regrid_compact_equals_full_flags(name):
    cfg = W.quadrant(N=128, n=16, levels=3, seed=1) if name == "quadrant" else W.shock_bubble(Nx=256, Ny=128, n=16, levels=3)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    a, b = amr.Mesh(cfg), amr.Mesh(cfg)
    a.set_state(fn)
    b.set_state(fn)
    seen_r = seen_c = 0
    n = cfg["n"]
    flat = np.zeros((4, n, n))
    flat[0], flat[3] = 1.0, 2.5
    for it in range(12):
        ref, crs = _own_requests(b)
        rb = b.regrid_with_requests(ref, crs)
        ra = a.regrid()
        assert ra == rb, (it, ra, rb)
        seen_r += ra[0]
        seen_c += ra[1]
        sa, sb = a.get_state(), b.get_state()
        assert set(sa) == set(sb), it
        for k in sa:
            assert np.array_equal(sa[k], sb[k]), (it, k)
        if it < 2:   # A28 init protocol: re-apply the initial condition on the refined mesh
            a.set_state(fn)
            b.set_state(fn)
        elif it >= 9:   # a uniform state: every sibling group of leaves becomes a coarsening request
            a.set_state(lambda l, P, Q: flat)
            b.set_state(lambda l, P, Q: flat)
        else:
            for _ in range(3):
                d1 = a.step(cfl=0.5)
                d2 = b.step(cfl=0.5)
                assert d1 == d2
    assert seen_r > 0 and seen_c > 0, (seen_r, seen_c)
