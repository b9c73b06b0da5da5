"""N > 1 host logic on CPU: two gloo ranks each compute their multi-rank plan through libamr.so's host-only
planning API (include/amr_debug.h) and check it against each other and against an independent statement of
what every rank's kernels read.  No GPU is touched."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2508_05020_b200 as amr
from paper_2508_05020_b200 import build as B

MOORE = [(0, 1), (1, 0), (0, -1), (-1, 0), (1, 1), (1, -1), (-1, -1), (-1, 1)]
SIDES = [(-1, 0), (1, 0), (0, -1), (0, 1)]


def _lib():
    B.build()
    L = amr.load()
    L.amr_plan_create.argtypes = [C.POINTER(amr.amr_config), C.POINTER(C.c_void_p)]
    L.amr_plan_destroy.argtypes = [C.c_void_p]
    L.amr_plan_destroy.restype = None
    L.amr_plan_regrid.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_uint8)]
    L.amr_plan_tree.argtypes = [C.c_void_p, C.c_int32, C.POINTER(amr.amr_patch_desc), C.c_int32,
                                C.POINTER(C.c_int32)]
    I = C.POINTER(C.c_int32)
    L.amr_plan_exchange.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, I, I, I, I, C.c_int32]
    return L


class Plan:
    def __init__(self, cfg):
        self.L = _lib()
        c = amr.make_config(cfg)
        self.h = C.c_void_p()
        assert self.L.amr_plan_create(C.byref(c), C.byref(self.h)) == 0

    def tree(self, world):
        cnt = C.c_int32()
        self.L.amr_plan_tree(self.h, world, None, 0, C.byref(cnt))
        arr = (amr.amr_patch_desc * cnt.value)()
        assert self.L.amr_plan_tree(self.h, world, arr, cnt.value, C.byref(cnt)) == 0
        return list(arr)

    def refine(self, keys):
        pos = {(d.level, d.i, d.j): e for e, d in enumerate(self.tree(1))}
        idx = np.array([pos[k] for k in keys], np.int32)
        bits = np.ones(len(keys), np.uint8)
        rc = self.L.amr_plan_regrid(self.h, len(keys), idx.ctypes.data_as(C.POINTER(C.c_int32)),
                                    bits.ctypes.data_as(C.POINTER(C.c_uint8)))
        assert rc == 0

    def exchange(self, world, rank, kind):
        cap = 1 << 16
        sc, rc_ = np.zeros(world, np.int32), np.zeros(world, np.int32)
        si, ri = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
        P = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))   # noqa: E731
        assert self.L.amr_plan_exchange(self.h, world, rank, kind, P(sc), P(si), P(rc_), P(ri), cap) == 0
        send, recv, o1, o2 = {}, {}, 0, 0
        for q in range(world):
            send[q] = si[o1:o1 + sc[q]].tolist(); o1 += sc[q]
            recv[q] = ri[o2:o2 + rc_[q]].tolist(); o2 += rc_[q]
        return send, recv


def amr_mesh_cfg():
    return dict(lo=(0.0, 0.0), hi=(1.0, 1.0), base=(128, 64), n=8, levels=3,
                bc=("periodic", "periodic", "reflective", "reflective"), scheme="weno5", ic="uniform")


def build_plan():
    p = Plan(amr_mesh_cfg())
    p.refine([(0, 3, 2), (0, 4, 2), (0, 9, 5), (0, 15, 7), (0, 0, 0)])
    p.refine([(1, 7, 5), (1, 18, 10)])
    return p


def needed_sources(tree, rank, world_tree):
    """Independent statement: remote tree indices read by the kernels of `rank`'s leaves."""
    key = {(d.level, d.i, d.j): e for e, d in enumerate(world_tree)}
    npx = {l: (128 // 8) << l for l in range(3)}
    npy = {l: (64 // 8) << l for l in range(3)}
    need = set()

    def pos(l, i, j):
        i %= npx[l]
        if j < 0 or j >= npy[l]:
            return None
        return key.get((l, i, j))

    for e, d in enumerate(world_tree):
        if not d.leaf or d.owner != rank:
            continue
        for dx, dy in SIDES:
            q = pos(d.level, d.i + dx, d.j + dy)
            if q is not None:
                if world_tree[q].owner != rank:
                    need.add(q)
            elif 0 <= d.j + dy < npy[d.level]:           # C/F side: parent's 3x3 neighbourhood
                P, Q = d.i // 2, d.j // 2
                for ddy in (-1, 0, 1):
                    for ddx in (-1, 0, 1):
                        c = pos(d.level - 1, P + ddx, Q + ddy)
                        if c is not None and world_tree[c].owner != rank:
                            need.add(c)
    return need


def needed_bands(tree, rank, world_tree, n=8):
    """Independent statement of the halo's band items (tree index * 32 + code): of a remote face neighbour the
    4-wide strip facing the reader (W neighbour: its columns n-4..n-1 = code 17; E: columns 0..3 = 16; S: its top
    row band n/4 - 1; N: its bottom row band 0), of a remote coarse source of a C/F side every row band (whole)."""
    key = {(d.level, d.i, d.j): e for e, d in enumerate(world_tree)}
    npx = {l: (128 // 8) << l for l in range(3)}
    npy = {l: (64 // 8) << l for l in range(3)}
    facing = {(-1, 0): 17, (1, 0): 16, (0, -1): n // 4 - 1, (0, 1): 0}
    need = set()

    def pos(l, i, j):
        i %= npx[l]
        if j < 0 or j >= npy[l]:
            return None
        return key.get((l, i, j))

    for d in world_tree:
        if not d.leaf or d.owner != rank:
            continue
        for dx, dy in SIDES:
            q = pos(d.level, d.i + dx, d.j + dy)
            if q is not None:
                if world_tree[q].owner != rank:
                    need.add(q * 32 + facing[(dx, dy)])
            elif 0 <= d.j + dy < npy[d.level]:
                for ddy in (-1, 0, 1):
                    for ddx in (-1, 0, 1):
                        c = pos(d.level - 1, d.i // 2 + ddx, d.j // 2 + ddy)
                        if c is not None and world_tree[c].owner != rank:
                            need.update(c * 32 + b for b in range(n // 4))
    return need


def needed_subcycle(tree, rank, levels=3):
    """Independent statement of the subcycled exchanges of `rank`: per level, remote same-level face
    neighbours of every owned active patch, remote coarse sources of owned leaves' C/F sides, remote fine leaves
    on owned leaves' coarse C/F sides."""
    key = {(d.level, d.i, d.j): e for e, d in enumerate(tree)}
    npx = {l: (128 // 8) << l for l in range(levels)}
    npy = {l: (64 // 8) << l for l in range(levels)}
    face, coarse, facc = ([set() for _ in range(levels)] for _ in range(3))

    def pos(l, i, j):
        i %= npx[l]
        if j < 0 or j >= npy[l]:
            return None
        return key.get((l, i, j))

    for d in tree:
        if d.owner != rank:
            continue
        l = d.level
        for dx, dy in SIDES:
            q = pos(l, d.i + dx, d.j + dy)
            if q is not None:
                if tree[q].owner != rank:
                    face[l].add(q)
                if d.leaf and not tree[q].leaf:        # the two fine leaves of q along the shared face
                    for k in range(2):
                        fi = 2 * tree[q].i + (1 if dx == -1 else 0 if dx == 1 else k)
                        fj = 2 * tree[q].j + (1 if dy == -1 else 0 if dy == 1 else k)
                        f = key[(l + 1, fi, fj)]
                        if tree[f].owner != rank:
                            facc[l].add(f)
            elif d.leaf and 0 <= d.j + dy < npy[l]:
                for ddy in (-1, 0, 1):
                    for ddx in (-1, 0, 1):
                        c = pos(l - 1, d.i // 2 + ddx, d.j // 2 + ddy)
                        if c is not None and tree[c].owner != rank:
                            coarse[l].add(c)
    return face, coarse, facc


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = build_plan()
        tr = p.tree(world)
        halo = dict(zip(("send", "recv"), p.exchange(world, rank, 0)))
        bands = dict(zip(("send", "recv"), p.exchange(world, rank, 1000)))
        flux = dict(zip(("send", "recv"), p.exchange(world, rank, 1)))
        sub = {k: [dict(zip(("send", "recv"), p.exchange(world, rank, 2 + 3 * l + w))) for l in range(3)]
               for w, k in enumerate(("face", "coarse", "facc"))}
        ns = needed_subcycle(tr, rank)
        mine = {"rank": rank, "owner": [d.owner for d in tr], "halo": halo, "flux": flux, "sub": sub,
                "sub_need": {k: [sorted(x) for x in v] for k, v in zip(("face", "coarse", "facc"), ns)},
                "need": sorted(needed_sources(tr, rank, tr)), "bands": bands,
                "need_bands": sorted(needed_bands(tr, rank, tr)),
                "leaves": sum(1 for d in tr if d.leaf and d.owner == rank)}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        q.put(("ok", rank, allv))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put(("err", rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def gathered():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
    return res[0][2]


def test_gloo_ranks_agree_on_replicated_partition(gathered):
    a, b = gathered
    assert a["owner"] == b["owner"], "replicated trees must give the same partition on every rank"
    assert set(a["owner"]) == {0, 1}
    # leaf balance: Morton cut of roots weighted by leaves
    tot = a["leaves"] + b["leaves"]
    assert abs(a["leaves"] - b["leaves"]) <= 0.25 * tot


@pytest.mark.parametrize("kind", ["halo", "flux"])
def test_gloo_send_lists_match_peer_receive_lists(gathered, kind):
    a, b = gathered
    assert a[kind]["send"][1] == b[kind]["recv"][0]
    assert b[kind]["send"][0] == a[kind]["recv"][1]
    assert a[kind]["send"][0] == [] and a[kind]["recv"][0] == []


def test_gloo_halo_covers_every_remote_read(gathered):
    for r in gathered:
        other = 1 - r["rank"]
        got = set(r["halo"]["recv"][other])
        assert set(r["need"]) == got
        assert all(r["owner"][q] == other for q in got)


def test_gloo_halo_moves_only_the_strips_read(gathered):
    """The halo exchange moves band items: exactly the facing 4-wide strip of every remote face neighbour and whole
    patches only for remote coarse sources of C/F ghost strips; the sender's list is the receiver's."""
    a, b = gathered
    assert a["bands"]["send"][1] == b["bands"]["recv"][0] and b["bands"]["send"][0] == a["bands"]["recv"][1]
    for r in gathered:
        got = set(r["bands"]["recv"][1 - r["rank"]])
        assert got == set(r["need_bands"])
        codes = [x & 31 for x in got]
        assert any(c >= 16 for c in codes) and any(c < 16 for c in codes)
    # fewer cells than whole patches: 2 of the 8 x 8 patch's 4 bands-worth per strip
    whole = 2 * len(a["need"])          # n/4 = 2 row bands per whole patch at n = 8
    assert len(a["bands"]["recv"][1]) < whole


def test_single_rank_has_no_exchange():
    p = build_plan()
    for kind in (0, 1):
        send, recv = p.exchange(1, 0, kind)
        assert send == {0: []} and recv == {0: []}
    assert {d.owner for d in p.tree(1)} == {0}


def test_partition_weak_scaling_slabs():
    """D5w: 4096 x 4096N cells in 32^2 patches -> each rank owns one 4096^2 square (Morton cut)."""
    for world in (2, 4, 8):
        cfg = dict(lo=(0.0, 0.0), hi=(1.0, float(world)), base=(4096, 4096 * world), n=32, levels=1,
                   bc=("periodic",) * 4, scheme="central4", ic="uniform")
        p = Plan(cfg)
        tr = p.tree(world)
        for d in tr:
            assert d.owner == d.j // 128, (world, d.i, d.j, d.owner)
        send, recv = p.exchange(world, 0, 0)
        # the square of rank 0 needs one row of 128 patches from each y-neighbour
        assert sum(len(v) for v in recv.values()) == 256   # two rows of 128 (periodic in y)
        send, recv = p.exchange(world, 0, 1000)
        # ... and of each of them only the 4-row strip facing it: 256 bands of 4 x 32 cells (1/8 of the patches)
        items = [x for v in recv.values() for x in v]
        assert len(items) == 256 and all((x & 31) in (0, 7) for x in items)


@pytest.mark.parametrize("kind", ["face", "coarse", "facc"])
def test_gloo_subcycle_lists_match_and_cover_every_remote_read(gathered, kind):
    """Subcycling across ranks: per level, rank 0's sends are rank 1's receives and vice versa, and every
    rank receives exactly the remote slots its level-l kernels read (independent statement above)."""
    a, b = gathered
    nonempty = 0
    for l in range(3):
        assert a["sub"][kind][l]["send"][1] == b["sub"][kind][l]["recv"][0]
        assert b["sub"][kind][l]["send"][0] == a["sub"][kind][l]["recv"][1]
        for r in gathered:
            got = r["sub"][kind][l]["recv"][1 - r["rank"]]
            assert sorted(got) == r["sub_need"][kind][l], (kind, l, r["rank"])
            nonempty += len(got)
    assert nonempty > 0, kind
