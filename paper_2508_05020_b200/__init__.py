"""B200-native AMR compressible-Euler hot path of arXiv 2508.05020 -- Python binding.

Argument marshalling only: every step of the numerical path runs in the sm_100a
kernels of ``libamr.so`` behind the C ABI declared in ``include/amr.h``.  There is
no CPU fallback: importing works without a GPU (so the ABI can be inspected), but
creating a mesh needs the CUDA library and a device and raises otherwise.
PyTorch is used only for device memory (optional ``pool`` tensor), streams and
process groups (NCCL unique-id broadcast).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libamr.so")

AMR_OK, AMR_E_ARG, AMR_E_CONFIG, AMR_E_NONPHYSICAL, AMR_E_MESH, AMR_E_CAPACITY, AMR_E_CUDA, AMR_E_COMM, \
    AMR_E_STATE = range(9)
STATUS = {0: "AMR_OK", 1: "AMR_E_ARG", 2: "AMR_E_CONFIG", 3: "AMR_E_NONPHYSICAL", 4: "AMR_E_MESH",
          5: "AMR_E_CAPACITY", 6: "AMR_E_CUDA", 7: "AMR_E_COMM", 8: "AMR_E_STATE"}
BC = {"periodic": 0, "transmissive": 1, "reflective": 2}
SCHEME = {"central4": 0, "weno5": 1}
COARSEN = {"r2_exact": 0, "alg2_literal": 1}

# every symbol include/amr.h declares (checked by tests/test_abi.py)
ABI_VERSION = 5   # include/amr.h AMR_ABI_VERSION: the amr_config / amr_stats layouts below
ABI_SYMBOLS = ["amr_abi_version", "amr_default_config", "amr_query_pool_bytes", "amr_create", "amr_destroy",
               "amr_set_state", "amr_set_state_fn", "amr_get_state", "amr_set_state_device", "amr_get_state_device", "amr_step", "amr_steps", "amr_sync", "amr_get_flags",
               "amr_regrid", "amr_regrid_with_flags", "amr_get_patch_tree", "amr_diagnostics",
               "amr_set_kernel_timing", "amr_get_stats", "amr_reset_stats", "amr_nccl_unique_id",
               "amr_last_error"]


class amr_config(C.Structure):
    _fields_ = [("dim", C.c_int32), ("lo", C.c_double * 2), ("hi", C.c_double * 2),
                ("base_cells", C.c_int32 * 2), ("patch_cells", C.c_int32), ("num_levels", C.c_int32),
                ("ratio", C.c_int32), ("gamma", C.c_double), ("bc", C.c_int32 * 4), ("scheme", C.c_int32),
                ("weno_characteristic", C.c_int32), ("div_order", C.c_int32), ("weno_eps", C.c_double),
                ("refine_threshold", C.c_double), ("coarsen_fraction", C.c_double), ("coarsen_rule", C.c_int32),
                ("max_patches", C.c_int32), ("pool", C.c_void_p), ("pool_bytes", C.c_uint64),
                ("cuda_stream", C.c_void_p), ("device", C.c_int32), ("world_size", C.c_int32),
                ("rank", C.c_int32), ("nccl_unique_id", C.c_void_p), ("check_positivity", C.c_int32),
                ("use_graphs", C.c_int32), ("comm_backend", C.c_int32), ("stage_kernel", C.c_int32), ("subcycle", C.c_int32),
                ("halo_mode", C.c_int32), ("host_comm", C.c_void_p), ("peer_map", C.c_int32)]


HOST_ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p)
HOST_BARRIER = C.CFUNCTYPE(C.c_int32, C.c_void_p)


class amr_host_comm(C.Structure):
    _fields_ = [("allgather", HOST_ALLGATHER), ("barrier", HOST_BARRIER), ("user", C.c_void_p)]


def gloo_host_comm():
    """(allgather, barrier) over the default torch.distributed group (e.g. gloo) for comm_backend 2: several
    processes, possibly on one GPU, exchange through host memory and map each other's pools with CUDA IPC."""
    import torch
    import torch.distributed as dist
    ws = dist.get_world_size()

    def allgather(send, nbytes, recv, _user):
        try:
            src = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send)).copy()
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(ws)]
            dist.all_gather(outs, torch.from_numpy(src))
            dst = np.ctypeslib.as_array((C.c_uint8 * (nbytes * ws)).from_address(recv))
            for q in range(ws):
                dst[q * nbytes:(q + 1) * nbytes] = outs[q].numpy()
            return 0
        except Exception:   # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def barrier(_user):
        try:
            dist.barrier()
            return 0
        except Exception:   # noqa: BLE001
            return 1

    return allgather, barrier


class amr_patch_desc(C.Structure):
    _fields_ = [("level", C.c_int32), ("i", C.c_int32), ("j", C.c_int32), ("parent", C.c_int32),
                ("child", C.c_int32 * 4), ("nbr", C.c_int32 * 8), ("owner", C.c_int32),
                ("leaf", C.c_uint8), ("refine_req", C.c_uint8), ("coarsen_req", C.c_uint8),
                ("ambiguous", C.c_uint8)]


class amr_stats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("stage_launches", C.c_int64), ("stage_ms", C.c_double),
                ("stage_timed", C.c_int64), ("stage_cells", C.c_int64), ("stage_bytes", C.c_double),
                ("steps", C.c_int64), ("leaf_cells", C.c_int64), ("leaves", C.c_int64), ("patches", C.c_int64),
                ("proxies", C.c_int64), ("sim_time", C.c_double)]


_lib = None
_P = C.c_void_p
IC_FN = C.CFUNCTYPE(None, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_U8 = C.POINTER(C.c_uint8)


def load(path: str = LIB_PATH):
    """Load libamr.so (build it first with ``python -m paper_2508_05020_b200.build``); raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA library {path} is missing: run `python -m paper_2508_05020_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(path)
    L.amr_abi_version.restype = C.c_int32
    if L.amr_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{path}: ABI version {L.amr_abi_version()} != {ABI_VERSION} (rebuild the library)")
    L.amr_default_config.argtypes = [C.POINTER(amr_config)]
    L.amr_query_pool_bytes.argtypes = [C.POINTER(amr_config), C.POINTER(C.c_uint64)]
    L.amr_create.argtypes = [C.POINTER(amr_config), C.POINTER(_P)]
    L.amr_destroy.argtypes = [_P]
    L.amr_destroy.restype = None
    L.amr_set_state.argtypes = [_P, C.c_int32, _I32, _D]
    L.amr_set_state_fn.argtypes = [_P, IC_FN, C.c_void_p]
    L.amr_get_state.argtypes = [_P, C.c_int32, _I32, _D]
    L.amr_set_state_device.argtypes = [_P, C.c_int32, _I32, C.c_void_p]
    L.amr_get_state_device.argtypes = [_P, C.c_int32, _I32, C.c_void_p]
    L.amr_step.argtypes = [_P, C.c_double, C.c_double, _D]
    L.amr_steps.argtypes = [_P, C.c_int32, C.c_double, C.c_double]
    L.amr_sync.argtypes = [_P]
    L.amr_get_flags.argtypes = [_P, C.c_int32, _D, _U8]
    L.amr_regrid.argtypes = [_P, _I32, _I32]
    L.amr_regrid_with_flags.argtypes = [_P, C.c_int32, _I32, _U8, _I32, _I32]
    L.amr_get_patch_tree.argtypes = [_P, C.POINTER(amr_patch_desc), C.c_int32, _I32]
    L.amr_diagnostics.argtypes = [_P, _D, _D]
    L.amr_set_kernel_timing.argtypes = [_P, C.c_int32]
    L.amr_get_stats.argtypes = [_P, C.POINTER(amr_stats)]
    L.amr_reset_stats.argtypes = [_P]
    L.amr_last_error.argtypes = [_P]
    L.amr_last_error.restype = C.c_char_p
    L.amr_nccl_unique_id.argtypes = [C.c_void_p]
    _lib = L
    return L


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (call on rank 0, broadcast to the others)."""
    buf = C.create_string_buffer(128)
    rc = load().amr_nccl_unique_id(buf)
    if rc != AMR_OK:
        raise AmrError(rc, "amr_nccl_unique_id failed (is torch's NCCL loadable?)")
    return buf.raw


class AmrError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def make_config(cfg: dict, **over) -> amr_config:
    """Marshal a workload dict (see workloads/) into the ABI's amr_config."""
    L = load()
    c = amr_config()
    L.amr_default_config(C.byref(c))
    c.dim = int(cfg.get("dim", 2))
    c.lo[0], c.lo[1] = cfg["lo"]
    c.hi[0], c.hi[1] = cfg["hi"]
    c.base_cells[0], c.base_cells[1] = cfg["base"]
    c.patch_cells = cfg["n"]
    c.num_levels = cfg["levels"]
    c.ratio = 2
    c.gamma = cfg.get("gamma", 1.4)
    for e, b in enumerate(cfg["bc"]):
        c.bc[e] = BC[b]
    c.scheme = SCHEME[cfg["scheme"]]
    c.weno_characteristic = int(cfg.get("characteristic", 1))
    c.div_order = int(cfg.get("div_order", 4))
    c.weno_eps = cfg.get("weno_eps", 1e-6)
    c.refine_threshold = cfg.get("theta", 0.1)
    c.coarsen_fraction = cfg.get("coarsen_frac", 0.25)
    c.coarsen_rule = COARSEN[cfg.get("coarsen_rule", "r2_exact")]
    roots = (cfg["base"][0] // cfg["n"]) * (cfg["base"][1] // cfg["n"])
    full = sum(4 ** l for l in range(cfg["levels"]))          # every root refined to the finest level
    c.max_patches = int(cfg.get("max_patches", max(16, roots * full)))
    c.check_positivity = int(cfg.get("check_positivity", 1))
    c.stage_kernel = int(cfg.get("stage_kernel", 0))
    c.use_graphs = int(cfg.get("use_graphs", 0))
    c.subcycle = int(cfg.get("subcycle", 0))
    c.halo_mode = int(cfg.get("halo_mode", 0))
    c.peer_map = int(cfg.get("peer_map", 0))
    c.world_size = 1
    c.rank = 0
    c.device = -1
    for k, v in over.items():
        setattr(c, k, v)
    return c


class Mesh:
    """One composite AMR mesh on one GPU (one rank), advanced by the CUDA path."""

    def __init__(self, cfg: dict, stream=None, pool=None, world_size=1, rank=0, comm_backend=0, comm_id=None,
                 **over):
        """world_size > 1: comm_backend 0 (NCCL; comm_id = 128-byte ncclUniqueId from nccl_unique_id(),
        broadcast by the caller), 1 (in-process loopback, one host thread per virtual rank; comm_id = group key)
        or 2 (one process per rank with host collectives; comm_id = (allgather, barrier), default
        gloo_host_comm() over torch.distributed)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2508_05020_b200.Mesh needs a CUDA device (no CPU fallback)")
        self.L = load()
        self.cfg = dict(cfg)
        self.n = cfg["n"]
        self._keep = []
        self.world_size, self.rank = world_size, rank
        if world_size > 1 and comm_backend == 2:   # host collectives (comm_id = (allgather, barrier) callables)
            ag, bar = comm_id if comm_id is not None else gloo_host_comm()
            hc = amr_host_comm(HOST_ALLGATHER(ag), HOST_BARRIER(bar), None)
            self._keep.append(hc)
            over.update(world_size=world_size, rank=rank, comm_backend=2,
                        host_comm=C.cast(C.pointer(hc), C.c_void_p).value)
        elif world_size > 1:
            key = comm_id if isinstance(comm_id, (bytes, bytearray)) else str(comm_id).encode()
            buf = C.create_string_buffer(bytes(key).ljust(128, b"\0")[:128], 128)
            self._keep.append(buf)
            over.update(world_size=world_size, rank=rank, comm_backend=comm_backend,
                        nccl_unique_id=C.cast(buf, C.c_void_p).value)
        if stream is None:
            stream = torch.cuda.current_stream()
        if stream.cuda_stream == 0:
            # the legacy default stream cannot be named through the ABI (NULL = library stream):
            # give the mesh its own torch stream so events recorded on `mesh.stream` bracket its kernels
            stream = torch.cuda.Stream()
        self.stream = stream
        over.setdefault("cuda_stream", stream.cuda_stream)
        over.setdefault("device", torch.cuda.current_device())
        c = make_config(cfg, **over)
        if pool == "torch":
            need = C.c_uint64()
            self.L.amr_query_pool_bytes(C.byref(c), C.byref(need))
            t = torch.empty(int(need.value), dtype=torch.uint8, device="cuda")
            self._keep.append(t)
            c.pool = t.data_ptr()
            c.pool_bytes = need.value
        self._c = c
        h = _P()
        rc = self.L.amr_create(C.byref(c), C.byref(h))
        if rc != AMR_OK:
            raise AmrError(rc, "amr_create failed (see stderr)")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.amr_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _chk(self, rc):
        if rc != AMR_OK:
            raise AmrError(rc, self.L.amr_last_error(self.h).decode())

    # ---- tree
    def tree(self):
        cnt = C.c_int32()
        self.L.amr_get_patch_tree(self.h, None, 0, C.byref(cnt))
        arr = (amr_patch_desc * max(1, cnt.value))()
        self._chk(self.L.amr_get_patch_tree(self.h, arr, cnt.value, C.byref(cnt)))
        return arr[:cnt.value]

    def keys(self):
        return [(d.level, d.i, d.j) for d in self.tree()]

    def leaves(self):
        return [(d.level, d.i, d.j) for d in self.tree() if d.leaf]

    # ---- state
    def owned(self):
        """Tree indices of the patches this rank owns (all of them on one rank)."""
        return np.array([e for e, d in enumerate(self.tree()) if d.owner == self.rank], np.int32)

    def set_state(self, fn=None, U=None, indices=None):
        """Set patches from fn(l, P, Q) -> U[4][n][n] (only the patches this rank owns are evaluated), or from
        U[k][4][n][n] for tree indices `indices` (default: every patch, tree order)."""
        if U is None:
            tr = self.tree()
            indices = self.owned() if indices is None else np.asarray(indices, np.int32)
            U = np.empty((len(indices), 4, self.n, self.n))
            for e, ti in enumerate(indices):
                d = tr[ti]
                U[e] = fn(d.level, d.i, d.j)
        if indices is None:
            indices = np.arange(len(self.tree()), dtype=np.int32)
        idx = np.ascontiguousarray(indices, dtype=np.int32)
        U = np.ascontiguousarray(U, dtype=np.float64)
        assert U.shape[0] == len(idx)
        self._chk(self.L.amr_set_state(self.h, len(idx), idx.ctypes.data_as(_I32), U.ctypes.data_as(_D)))

    def set_state_points(self, fn):
        """Set every owned patch through the C callback amr_set_state_fn: fn(x, y) -> (rho, rho u, rho v, rho e)
        arrays at the given cell centres (x, y: 1D float64 arrays of one patch's n^2 points)."""
        def cb(ncell, x, y, U, _user):
            xs = np.ctypeslib.as_array(x, shape=(ncell,))
            ys = np.ctypeslib.as_array(y, shape=(ncell,))
            out = np.ctypeslib.as_array(U, shape=(4 * ncell,))
            out[:] = np.asarray(fn(xs, ys), dtype=np.float64).reshape(-1)
        c_cb = IC_FN(cb)   # kept alive for the duration of the call
        self._chk(self.L.amr_set_state_fn(self.h, c_cb, None))

    def set_state_device(self, tensor, indices=None):
        """Set patches (default: every patch, tree order) from a contiguous CUDA float64 tensor [k][4][n][n]."""
        idx = np.arange(len(self.tree()), dtype=np.int32) if indices is None else np.asarray(indices, np.int32)
        assert tensor.is_cuda and tensor.dtype.is_floating_point and tensor.is_contiguous()
        assert tensor.numel() == len(idx) * 4 * self.n * self.n
        self._chk(self.L.amr_set_state_device(self.h, len(idx), idx.ctypes.data_as(_I32), tensor.data_ptr()))

    def get_state_device(self, tensor, indices=None):
        idx = np.arange(len(self.tree()), dtype=np.int32) if indices is None else np.asarray(indices, np.int32)
        assert tensor.is_cuda and tensor.is_contiguous() and tensor.numel() == len(idx) * 4 * self.n * self.n
        self._chk(self.L.amr_get_state_device(self.h, len(idx), idx.ctypes.data_as(_I32), tensor.data_ptr()))

    def get_state(self, as_dict=True, indices=None, out=None):
        """State of patches `indices` (default all; on several ranks only owned patches are filled).  `out`: a
        preallocated C-contiguous float64 array [k][4][n][n] to fill (e.g. a pinned-memory view: the download
        then runs at full PCIe rate, with no fresh pageable allocation)."""
        tr = self.tree() if (as_dict or indices is None) else None
        idx = np.arange(len(tr), dtype=np.int32) if indices is None else np.ascontiguousarray(indices, np.int32)
        if out is None:
            U = np.empty((len(idx), 4, self.n, self.n))
        else:
            U = out
            assert U.dtype == np.float64 and U.flags.c_contiguous and U.size == len(idx) * 4 * self.n * self.n
        self._chk(self.L.amr_get_state(self.h, len(idx), idx.ctypes.data_as(_I32), U.ctypes.data_as(_D)))
        if not as_dict:
            return U
        return {(tr[ti].level, tr[ti].i, tr[ti].j): U[e] for e, ti in enumerate(idx)}

    # ---- stepping
    def step(self, dt=0.0, cfl=0.0, want_dt=True):
        d = C.c_double()
        self._chk(self.L.amr_step(self.h, float(dt), float(cfl), C.byref(d) if want_dt else None))
        return d.value if want_dt else None

    def steps(self, k, dt=0.0, cfl=0.0):
        self._chk(self.L.amr_steps(self.h, int(k), float(dt), float(cfl)))

    def sync(self):
        self._chk(self.L.amr_sync(self.h))

    # ---- AMR
    def flags(self):
        tr = self.tree()
        m = len(tr)
        me = np.zeros(m)
        bits = np.zeros(m, np.uint8)
        self._chk(self.L.amr_get_flags(self.h, m, me.ctypes.data_as(_D), bits.ctypes.data_as(_U8)))
        return {(d.level, d.i, d.j): (float(me[e]), bool(bits[e] & 1), bool(bits[e] & 2), bool(bits[e] & 4))
                for e, d in enumerate(tr)}

    def regrid(self):
        nr, nc = C.c_int32(), C.c_int32()
        self._chk(self.L.amr_regrid(self.h, C.byref(nr), C.byref(nc)))
        return nr.value, nc.value

    def regrid_with_requests(self, refine_keys=(), coarsen_keys=()):
        pos = {k: e for e, k in enumerate(self.keys())}
        keys = sorted(set(refine_keys) | set(coarsen_keys))
        rs, cs = set(refine_keys), set(coarsen_keys)
        idx = np.array([pos[k] for k in keys], np.int32)
        bits = np.array([(k in rs) | ((k in cs) << 1) for k in keys], np.uint8)
        nr, nc = C.c_int32(), C.c_int32()
        self._chk(self.L.amr_regrid_with_flags(self.h, len(keys), idx.ctypes.data_as(_I32),
                                               bits.ctypes.data_as(_U8), C.byref(nr), C.byref(nc)))
        return nr.value, nc.value

    # ---- diagnostics
    def diagnostics(self):
        t = np.zeros(4)
        lam = C.c_double()
        self._chk(self.L.amr_diagnostics(self.h, t.ctypes.data_as(_D), C.byref(lam)))
        return t, lam.value

    def set_kernel_timing(self, on=True):
        self._chk(self.L.amr_set_kernel_timing(self.h, int(on)))

    def stats(self):
        s = amr_stats()
        self._chk(self.L.amr_get_stats(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in amr_stats._fields_}

    def reset_stats(self):
        self._chk(self.L.amr_reset_stats(self.h))
