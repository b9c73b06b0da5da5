"""Multi-PROCESS data path on one GPU: 2 processes (torch.multiprocessing + gloo) each own one rank of the mesh
(comm_backend 2: host collectives over gloo, peer pools mapped with real CUDA IPC between the processes).  This
exercises what the in-process loopback cannot: cudaIpcGetMemHandle / cudaIpcOpenMemHandle of another process's
pool, the peer-pull kernel and the stage kernel's TMA loads reading IPC-mapped memory (halo_mode 1 / 2), and the
cross-process fence (stream synchronise + host barrier; no kernel ever waits on another process).  The owned
results must be bitwise those of one rank, which is itself run in lockstep with the oracle (1e-11)."""
import os
import socket

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

CASES = {
    "uniform_c4_n32": (W.sweep(N=256, n=32, scheme="central4", seed=3, ic="smooth"), 3, None),
    "implosion_c4_amr_n32": (W.implosion(N=256, n=32, scheme="central4", levels=2), 4, 2),
    "quadrant_weno_amr": (W.quadrant(N=64, n=16, levels=3, seed=2), 6, 3),
    "noise_c4_n32": (dict(W.sweep(N=256, n=32, scheme="central4", Ny=512, seed=7), check_positivity=0, cfl=0.3), 2, None),
}


def _drive(g, cfg, steps, regrid):
    fn = lambda l, P, Q: W.patch_state(cfg, l, P, Q)   # noqa: E731
    g.set_state(fn)
    for _ in range(cfg["levels"] - 1):
        g.regrid()
        g.set_state(fn)
    dts = []
    for s in range(1, steps + 1):
        dts.append(g.step(cfl=cfg.get("cfl", 0.5)))
        if regrid and s % regrid == 0:
            g.regrid()
    return dts


def _worker(rank, world, port, name, halo_mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import paper_2508_05020_b200 as amr
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg, steps, regrid = CASES[name]
        g = amr.Mesh(dict(cfg, halo_mode=halo_mode), world_size=world, rank=rank, comm_backend=2)
        dts = _drive(g, cfg, steps, regrid)
        tree = g.tree()
        st = g.get_state()
        owned = {(d.level, d.i, d.j) for d in tree if d.owner == rank}
        q.put(("ok", rank, {k: v for k, v in st.items() if k in owned}, g.keys(), dts))
        g.close()
    except Exception as e:   # pragma: no cover - surfaced by the parent
        q.put(("err", rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("name,halo_mode", [("uniform_c4_n32", 0), ("uniform_c4_n32", 1), ("uniform_c4_n32", 2),
                                            ("implosion_c4_amr_n32", 2), ("quadrant_weno_amr", 1),
                                            ("quadrant_weno_amr", 2),
                                            ("noise_c4_n32", 0), ("noise_c4_n32", 2)])
def test_two_processes_bitwise_equal_single_rank(name, halo_mode):
    import torch.multiprocessing as mp
    import paper_2508_05020_b200 as amr
    from tests.parity import run_pair
    cfg, steps, regrid = CASES[name]
    stats = {}
    o, g, e = run_pair(cfg, steps, cfl=cfg.get("cfl", 0.5), regrid_every=regrid, stats=stats)
    assert e <= 1e-11
    ref_dts = stats["dts"]
    ref, ref_keys = g.get_state(), g.keys()
    g.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, halo_mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    merged = {}
    for tag, r, st, keys, dts in res:
        assert tag == "ok", (r, st)
        assert keys == ref_keys and dts == ref_dts, r
        merged.update(st)
    assert set(merged) == set(ref)
    for k, U in ref.items():
        assert np.array_equal(U, merged[k]), (name, halo_mode, k)
