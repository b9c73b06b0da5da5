"""GPU parity: the CUDA path through the C ABI against the oracle, element by element (1e-11, O18), trees and
flags in lockstep (A32).  Sizes span several tiles/patches with ragged level structure; full-size configs are
checked on sampled patches (test_gpu_fullsize.py)."""
import numpy as np
import pytest

import oracle as orc
import paper_2508_05020_b200 as amr
import workloads as W
from tests.parity import parity_error, run_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [8, 16, 32, 64])
def test_vortex_central4_uniform(n):
    """BJ configs[1] scaled to 128^2 (256^2 for n = 64 so there are several patches): 10 CFL-0.5 steps."""
    N = 256 if n == 64 else 128
    run_pair(W.vortex(N=N, n=n), steps=10, cfl=0.5)


@pytest.mark.parametrize("char", [1, 0])
def test_vortex_weno_uniform(char):
    run_pair(W.vortex(N=128, n=32, scheme="weno5", characteristic=char), steps=10, cfl=0.5)


@pytest.mark.parametrize("div", [2, 4])
@pytest.mark.parametrize("scheme", ["central4", "weno5"])
def test_divergence_orders(scheme, div):
    run_pair(W.vortex(N=64, n=16, scheme=scheme, div_order=div), steps=5, cfl=0.4)


@pytest.mark.parametrize("seed", [1, 2])
def test_quadrant_amr_lockstep(seed):
    """BJ configs[2] at 64^2 base, 3 levels, 16^2 patches, transmissive, WENO5-char, regrid every 4 steps."""
    cfg = W.quadrant(N=64, n=16, levels=3, seed=seed)
    stats = {}
    o, g, e = run_pair(cfg, steps=10, cfl=0.5, regrid_every=4, stats=stats)
    levels = {k[0] for k in g.leaves()}
    assert len(levels) >= 2


def test_sod_strip_two_levels():
    """BJ configs[0] (A21/A23): 13 roots of 16^2, transmissive x, periodic y (dim = 1 strip), 2 levels."""
    cfg = dict(W.sod(), dim=1)
    run_pair(cfg, steps=10, cfl=0.5, regrid_every=4)


def test_shock_bubble_reflective_amr():
    """BJ configs[3] at 128x64 base, 3 levels: reflective walls (mirror + negated normal momentum)."""
    cfg = W.shock_bubble(Nx=128, Ny=64, n=16, levels=3)
    run_pair(cfg, steps=10, cfl=0.5, regrid_every=4)


def test_blast_periodic_amr_component_weno():
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(64, 64), n=8, levels=3, bc=("periodic",) * 4,
               scheme="weno5", characteristic=0, div_order=4, ic="blast", blast_width=0.08, theta=0.02,
               coarsen_frac=0.25, weno_eps=1e-6, gamma=1.4, cfl=0.4)
    run_pair(cfg, steps=10, regrid_every=4, check_each=True)


def test_free_stream_bitwise_gpu_amr():
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(32, 32), n=8, levels=3,
               bc=("transmissive", "transmissive", "reflective", "reflective"), scheme="weno5", characteristic=1,
               div_order=4, ic="uniform", uniform_state=(1.3, 0.4, 0.0, 0.9))
    g = amr.Mesh(cfg)
    g.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    g.regrid_with_requests([(0, 1, 1), (0, 2, 1), (0, 0, 3)])
    g.regrid_with_requests([(1, 3, 3), (1, 2, 2)])
    g.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    before = g.get_state()
    for _ in range(3):
        g.step(cfl=0.5)
    after = g.get_state()
    for k in before:
        assert np.array_equal(before[k], after[k]), k


def test_conservation_gpu_periodic_amr():
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(64, 64), n=16, levels=3, bc=("periodic",) * 4,
               scheme="weno5", characteristic=1, div_order=4, ic="blast", blast_width=0.08, theta=0.02,
               coarsen_frac=0.25, weno_eps=1e-6, gamma=1.4)
    g = amr.Mesh(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    g.set_state(fn)
    for _ in range(2):
        g.regrid()
        g.set_state(fn)
    t0, _ = g.diagnostics()
    st = g.get_state()
    scale = sum(np.abs(U).sum(axis=(1, 2)) * (1.0 / (64 << l)) ** 2 for (l, P, Q), U in st.items()
                if (l, P, Q) in set(g.leaves()))
    for s in range(1, 11):
        g.step(cfl=0.4)
        if s % 4 == 0:
            g.regrid()
    t1, _ = g.diagnostics()
    assert np.all(np.abs(t1 - t0) <= 1e-12 * scale), (t1 - t0) / scale


@pytest.mark.parametrize("variant", [1, 0])
@pytest.mark.parametrize("scheme", ["central4", "weno5"])
def test_patch_size_invariance_bitwise(scheme, variant):
    """on a uniform periodic mesh the decomposition is invisible: n = 8/16/32/64 give bitwise-equal states
    when the same kernel arithmetic runs (stage_kernel 1, and every WENO path).  With the default Central4 kernel,
    n = 32/64 run the TMA kernel (its RK sums are ordered W = U + dt Lx, then + dt Ly): bitwise among themselves,
    equal to rounding against n = 8/16."""
    res = {}
    for n in (8, 16, 32, 64):
        cfg = W.sweep(N=128, n=n, scheme=scheme, seed=3, stage_kernel=variant)
        cfg["ic"] = "smooth"
        g = amr.Mesh(cfg)
        U0 = W.level0_state(cfg)
        g.set_state(U=U0.reshape(-1, 4, n, n))
        for _ in range(3):
            g.step(dt=1e-5)
        U = g.get_state(as_dict=False).reshape(128 // n, 128 // n, 4, n, n).transpose(2, 0, 3, 1, 4).reshape(4, 128, 128)
        res[n] = U
    assert np.array_equal(res[8], res[16])
    assert np.array_equal(res[32], res[64])
    if scheme == "weno5" or variant == 1:
        assert np.array_equal(res[8], res[32])
    else:
        scale = np.abs(res[8]).max(axis=(1, 2), keepdims=True)
        assert np.max(np.abs(res[8] - res[32]) / scale) <= 1e-14


def test_single_root_periodic_self_neighbour():
    """a 1x1 periodic scaffold is its own neighbour in all 8 directions."""
    cfg = W.vortex(N=32, n=32, L=10.0)
    g = amr.Mesh(cfg)
    d = g.tree()[0]
    assert list(d.nbr) == [0] * 8
    run_pair(cfg, steps=3, cfl=0.5)


def test_nonphysical_step_not_committed():
    cfg = W.sweep(N=64, n=16, scheme="central4", seed=5)
    g = amr.Mesh(cfg)
    U0 = W.level0_state(cfg).reshape(-1, 4, 16, 16).copy()
    U0[5, 0, 3, 3] = -1.0            # negative density
    g.set_state(U=U0)
    before = g.get_state(as_dict=False)
    with pytest.raises(amr.AmrError) as ei:
        g.step(dt=1e-4)
    assert ei.value.code == amr.AMR_E_NONPHYSICAL
    assert "stage" in str(ei.value)
    assert np.array_equal(before, g.get_state(as_dict=False))


def test_steps_report_a_nonphysical_state_late_without_rollback():
    """include/amr.h amr_steps: a non-physical state in a batch is reported by the next amr_sync (AMR_E_NONPHYSICAL),
    and the mesh keeps the advanced state (no rollback, unlike amr_step)."""
    cfg = W.sweep(N=64, n=16, scheme="central4", seed=5)
    g = amr.Mesh(cfg)
    U0 = W.level0_state(cfg).reshape(-1, 4, 16, 16).copy()
    U0[5, 0, 3, 3] = -1.0
    g.set_state(U=U0)
    before = g.get_state(as_dict=False)
    g.steps(3, dt=1e-4)              # queued: no error yet
    with pytest.raises(amr.AmrError) as ei:
        g.sync()
    assert ei.value.code == amr.AMR_E_NONPHYSICAL
    assert not np.array_equal(before, g.get_state(as_dict=False))
    assert g.stats()["steps"] == 3


def test_capacity_error_leaves_mesh_unchanged():
    cfg = dict(W.quadrant(N=64, n=16, levels=3), max_patches=20)
    g = amr.Mesh(cfg)
    g.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    keys = g.keys()
    with pytest.raises(amr.AmrError) as ei:
        g.regrid_with_requests([(0, 1, 1), (0, 2, 2)])
    assert ei.value.code == amr.AMR_E_CAPACITY
    assert g.keys() == keys
    g.step(cfl=0.5)


def test_tree_matches_oracle_after_random_requests():
    cfg = dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(32, 32), n=8, levels=4, bc=("periodic",) * 4,
               scheme="central4", ic="uniform")
    rng = np.random.default_rng(0)
    o = orc.Oracle(cfg)
    g = amr.Mesh(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    o.set_state(fn)
    g.set_state(fn)
    for it in range(30):
        tr = o.tree()
        leaves = [(l, P, Q) for (l, P, Q, lf) in tr if lf and l < 3]
        parents = [(l, P, Q) for (l, P, Q, lf) in tr if not lf]
        ref = [leaves[i] for i in rng.choice(len(leaves), size=min(3, len(leaves)), replace=False)]
        crs = [parents[i] for i in rng.choice(len(parents), size=min(2, len(parents)), replace=False)] if parents else []
        assert o.regrid_with_requests(ref, crs) == g.regrid_with_requests(ref, crs)
        assert [(l, P, Q) for (l, P, Q, _) in o.tree()] == g.keys()
    e, _ = parity_error(o.get_state(), g.get_state())
    assert e == 0.0


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [8, 16, 32, 64])
def test_central4_amr_walls(n, variant):
    """Central4 on a 2-level mesh with C/F faces (proxies, flux registers, reflux) and transmissive / reflective
    walls, for every stage-kernel organisation: 0 = persistent TMA-pipelined (n >= 32; n = 8, 16: 32 x 32 blocks
    of leaves plus the per-tile kernel for leaves outside complete blocks), 1 = one CTA per tile,
    2 = unfused (four kernels, intermediates through HBM), 3 = one launch per leaf patch."""
    N = 256 if n == 64 else 128
    cfg = W.vortex(N=N, n=n, levels=2, theta=0.02 if n == 64 else 0.01, stage_kernel=variant,
                   bc=("transmissive", "transmissive", "reflective", "reflective"))
    o, g, e = run_pair(cfg, steps=10, cfl=0.5, regrid_every=4)
    assert len({k[0] for k in g.leaves()}) == 2


@pytest.mark.parametrize("div", [4, 2])
@pytest.mark.parametrize("n", [32, 64])
def test_stage_kernel_variants_agree(n, div):
    """The warp-specialised TMA kernel and the per-tile Central4 kernel evaluate the same scheme; they differ only
    in the order of the final RK sums (W = U + dt Lx, then + dt Ly): equal to rounding."""
    res = []
    for variant in (0, 1):
        cfg = W.sweep(N=256, n=n, scheme="central4", seed=11, stage_kernel=variant, check_positivity=0,
                      div_order=div)
        g = amr.Mesh(cfg)
        g.set_state(U=W.level0_state(cfg).reshape(-1, 4, n, n))
        for _ in range(3):
            g.step(dt=2e-6)
        res.append(g.get_state(as_dict=False))
    scale = np.abs(res[1]).max(axis=(0, 2, 3), keepdims=True)
    assert np.max(np.abs(res[0] - res[1]) / scale) <= 1e-13


@pytest.mark.parametrize("case", ["quadrant_amr", "vortex_c4"])
def test_cuda_graph_replay_bitwise(case):
    """use_graphs = 1 replays one captured step per RK-buffer position once a plan has served 3 steps (re-captured
    after each regrid): states, dt and trees bitwise equal to the stream-launched path, CFL and fixed-dt steps."""
    if case == "quadrant_amr":
        base = W.quadrant(N=64, n=16, levels=3, seed=2)
    else:
        base = W.vortex(N=128, n=32)
    runs = []
    for graphs in (0, 1):
        cfg = dict(base, use_graphs=graphs)
        g = amr.Mesh(cfg)
        fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
        g.set_state(fn)
        for _ in range(cfg["levels"] - 1):
            g.regrid()
            g.set_state(fn)
        dts = []
        for s in range(1, 15):
            dts.append(g.step(cfl=0.5) if s % 3 else g.step(dt=1e-4))
            if s % 7 == 0:
                g.regrid()
        st = g.stats()
        runs.append((g.get_state(), dts, g.keys()))
    (s0, d0, k0), (s1, d1, k1) = runs
    assert k0 == k1 and d0 == d1
    for key in s0:
        assert np.array_equal(s0[key], s1[key]), key


@pytest.mark.parametrize("scheme", ["central4", "weno5"])
def test_implosion_parity(scheme):
    """NEXT #2, Eq. 13 at 128^2 (32^2 patches, periodic, CFL 0.45): oracle parity over 10 steps."""
    run_pair(W.implosion(N=128, n=32, scheme=scheme), steps=10, cfl=0.45)


@pytest.mark.parametrize("scheme", ["central4", "weno5"])
def test_implosion_fullsize_symmetry(scheme):
    """Eq. 13 at the paper's 1024^2: after 20 CFL-0.45 steps the GPU state keeps the x <-> y and mirror
    symmetries of the IC (a property that holds at any size) and conserves the totals."""
    cfg = W.implosion(N=1024, n=32, scheme=scheme)
    g = amr.Mesh(cfg)
    g.set_state(U=W.level0_state(cfg).reshape(-1, 4, 32, 32))
    t0, _ = g.diagnostics()
    for _ in range(20):
        g.step(cfl=0.45)
    t1, _ = g.diagnostics()
    U = g.get_state(as_dict=False).reshape(32, 32, 4, 32, 32).transpose(2, 0, 3, 1, 4).reshape(4, 1024, 1024)
    scale = np.abs(U).reshape(4, -1).max(axis=1)
    T = U.transpose(0, 2, 1)[[0, 2, 1, 3]]
    M = U[:, :, ::-1].copy()
    M[1] = -M[1]
    for k in range(4):
        assert np.abs(U[k] - T[k]).max() <= 1e-12 * scale[k], ("transpose", k)
        assert np.abs(U[k] - M[k]).max() <= 1e-12 * scale[k], ("mirror", k)
    vol = np.abs(U).reshape(4, -1).sum(axis=1) * (0.6 / 1024) ** 2
    assert np.all(np.abs(t1 - t0) <= 1e-12 * vol)


@pytest.mark.parametrize("variant", [2, 3])
@pytest.mark.parametrize("char", [1, 0])
def test_weno_amr_unfused_and_per_patch(variant, char):
    """The NEXT #1 organisations on the WENO5 path with AMR (quadrant, 3 levels, regrids): oracle parity."""
    cfg = W.quadrant(N=64, n=16, levels=3, seed=1, stage_kernel=variant, characteristic=char)
    run_pair(cfg, steps=6, cfl=0.5, regrid_every=3)


def test_set_state_fn_matches_patch_arrays():
    """amr_set_state_fn samples the IC at cell centres (A33) through a C callback; on a 3-level mesh it equals
    set_state with the same IC evaluated per patch in numpy (workloads.patch_state)."""
    cfg = W.quadrant(N=64, n=16, levels=3, seed=2, ic="vortex", vortex_centre=(0.5, 0.5), hi=(1.0, 1.0))
    cfg["vortex_beta"] = 5.0
    g1 = amr.Mesh(cfg)
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    g1.set_state(fn)
    g1.regrid_with_requests([(0, 1, 1), (0, 2, 2)])
    g1.regrid_with_requests([(1, 3, 3)])
    g2 = amr.Mesh(cfg)
    g2.set_state(fn)
    g2.regrid_with_requests([(0, 1, 1), (0, 2, 2)])
    g2.regrid_with_requests([(1, 3, 3)])
    g1.set_state(fn)

    def pts(x, y):
        rho, u, v, p = W.vortex_prim(cfg, x, y)
        return W.to_conserved(rho, u, v, p, cfg["gamma"])
    g2.set_state_points(pts)
    s1, s2 = g1.get_state(), g2.get_state()
    assert set(s1) == set(s2)
    for k in s1:
        np.testing.assert_allclose(s2[k], s1[k], rtol=0, atol=1e-14 * np.abs(s1[k]).max())


def test_empty_calls():
    """Zero-patch state transfers and an empty request list are valid no-ops."""
    cfg = W.quadrant(N=64, n=16, levels=2, seed=3)
    g = amr.Mesh(cfg)
    g.set_state(lambda l, P, Q: W.patch_state(cfg, l, P, Q))
    before = g.get_state()
    g.set_state(U=np.zeros((0, 4, 16, 16)), indices=np.zeros(0, np.int32))
    assert g.get_state(as_dict=False, indices=np.zeros(0, np.int32)).shape == (0, 4, 16, 16)
    assert g.regrid_with_requests([], []) == (0, 0)
    after = g.get_state()
    assert set(before) == set(after) and all(np.array_equal(before[k], after[k]) for k in before)
    g.close()
