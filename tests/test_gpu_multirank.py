"""Multi-rank data path on ONE GPU: W virtual ranks (host threads, comm_backend = in-process loopback) run the
same mesh as one rank; the final states must be BITWISE identical (SURVEY.md s8(e) rank invariance) to the
single-rank run, which is itself run in lockstep with the oracle (tests/parity.run_pair: flags compared at
every regrid, the final state within 1e-11), so every multi-rank result is oracle-checked.  This exercises ownership, halo / flux-register / coarse-source exchanges, the
Lambda and flag collectives and patch migration at regrid with the real kernels; only the transport (NCCL vs
device-to-device copies) differs from the one-process-per-GPU path.  The virtual ranks never spin on each
other: every cross-rank dependency is a CUDA event between their streams."""
import threading
import uuid

import numpy as np
import pytest

import paper_2508_05020_b200 as amr
import workloads as W
from tests.parity import parity_error, run_pair

pytestmark = pytest.mark.gpu

_REF = {}


def run_single(cfg, steps, regrid_every):
    """One rank, in lockstep with the oracle (A28 init, A32 flags, 1e-11 at the end); cached per case."""
    key = (repr(sorted(cfg.items())), steps, regrid_every)
    if key not in _REF:
        stats = {}
        o, g, e = run_pair(cfg, steps, cfl=cfg.get("cfl", 0.5), regrid_every=regrid_every, stats=stats)
        assert e <= 1e-11
        _REF[key] = (g.get_state(), g.keys(), list(stats["dts"]))
        g.close()
    return _REF[key]


def run_multi(cfg, world, steps, regrid_every):
    key = uuid.uuid4().hex[:16]
    out = [None] * world
    err = []

    def worker(r):
        try:
            import torch
            torch.cuda.set_device(0)
            g = amr.Mesh(cfg, world_size=world, rank=r, comm_backend=1, comm_id=key)
            fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
            g.set_state(fn)
            for _ in range(cfg["levels"] - 1):
                g.regrid()
                g.set_state(fn)
            dts = []
            for s in range(1, steps + 1):
                dts.append(g.step(cfl=cfg.get("cfl", 0.5)))
                if regrid_every and s % regrid_every == 0:
                    g.regrid()
            tree = g.tree()
            st = g.get_state()
            owned = {(d.level, d.i, d.j) for d in tree if d.owner == r}
            out[r] = ({k: v for k, v in st.items() if k in owned}, g.keys(), dts,
                      {d.owner for d in tree}, g.stats())
            g.close()
        except Exception as e:   # surfaced below
            err.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    return out


CASES = {
    "uniform_periodic_c4_n32": (W.sweep(N=256, n=32, scheme="central4", seed=3, ic="smooth"), 4, None),
    "implosion_c4_amr_n32": (W.implosion(N=256, n=32, scheme="central4", levels=2), 6, 3),
    "uniform_periodic_c4": (W.sweep(N=128, n=16, scheme="central4", seed=3, ic="smooth"), 4, None),
    "quadrant_amr_weno": (W.quadrant(N=64, n=16, levels=3, seed=2), 8, 4),
    "shock_bubble_reflective": (W.shock_bubble(Nx=128, Ny=64, n=16, levels=3), 8, 4),
    "shock_bubble_subcycled": (dict(W.shock_bubble(Nx=128, Ny=64, n=16, levels=3), subcycle=1), 4, 2),
    "implosion_c4_amr_n16": (W.implosion(N=128, n=16, scheme="central4", levels=2), 6, 3),
    "implosion_c4_subcycled_n32": (W.implosion(N=256, n=32, scheme="central4", levels=3, subcycle=1), 4, 2),
}


@pytest.mark.parametrize("halo_mode", [0, 1, 2])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", list(CASES))
def test_virtual_ranks_bitwise_equal_single_rank(case, world, halo_mode):
    """halo_mode 0: pack + transport copy + unpack; 1: peer pull (NEXT #3) from the other ranks' mapped pools;
    2: the stage kernel loads remote face strips from the owners' pools itself (Central4 TMA kernel, n >= 32, and
    per-tile kernel, every n; WENO5 per-tile and n = 8 block-tile kernels)."""
    cfg, steps, regrid = CASES[case]
    if halo_mode == 2 and cfg["scheme"] == "central4" and cfg["n"] < 32:
        # the n = 8 / 16 block-tile kernels read block-edge strips from the local pool only: halo_mode 2 runs Central4
        # there on the per-tile kernel (stage_kernel 1), and so does the single-rank reference
        cfg = dict(cfg, stage_kernel=1)
    ref_state, ref_keys, ref_dts = run_single(cfg, steps, regrid)
    res = run_multi(dict(cfg, halo_mode=halo_mode), world, steps, regrid)
    merged = {}
    for r, (st, keys, dts, owners, stats) in enumerate(res):
        assert keys == ref_keys, f"rank {r}: tree differs"
        assert dts == ref_dts, f"rank {r}: dt sequence differs"
        assert owners == set(range(world)), f"rank {r}: not every rank owns patches"
        merged.update(st)
    assert set(merged) == set(ref_state)
    for k, U in ref_state.items():
        assert np.array_equal(U, merged[k]), (case, world, k)
    e, _ = parity_error(ref_state, merged)
    assert e == 0.0


def test_peer_pull_launches_one_kernel_per_exchange():
    """halo_mode 1 replaces the pack and unpack kernels of every halo / flux exchange by one pull kernel: on the
    same run it launches fewer kernels than halo_mode 0 and moves the same patch bytes."""
    cfg, steps, regrid = CASES["quadrant_amr_weno"]
    st = {}
    for hm in (0, 1):
        res = run_multi(dict(cfg, halo_mode=hm), 2, steps, regrid)
        st[hm] = res[0][4]
    assert st[1]["launches"] < st[0]["launches"], st


@pytest.mark.parametrize("halo_mode", [0, 1, 2])
def test_more_ranks_than_roots(halo_mode):
    """Degenerate partition: 6 virtual ranks over 4 root patches -- two ranks own nothing and run every
    collective with empty launch lists; the owned results are still bitwise those of one rank."""
    cfg = W.sweep(N=64, n=32, scheme="central4", seed=5, ic="smooth")
    ref_state, ref_keys, ref_dts = run_single(cfg, 3, None)
    res = run_multi(dict(cfg, halo_mode=halo_mode), 6, 3, None)
    merged = {}
    owners = set()
    for r, (st, keys, dts, own, stats) in enumerate(res):
        assert keys == ref_keys and dts == ref_dts
        owners |= {r} if st else set()
        merged.update(st)
    assert len(owners) == 4
    for k, U in ref_state.items():
        assert np.array_equal(U, merged[k]), k
