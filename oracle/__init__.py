"""CPU ORACLE of the AMR compressible-Euler hot path (arXiv 2508.05020).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with the CUDA product path
(``paper_2508_05020_b200``); neither imports the other.  The arithmetic lives
in ``oracle.cpp`` (plain C++17, fp64, ``-O2 -ffp-contract=off``); this module
only marshals arguments through ctypes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "oracle.cpp"), os.path.join(_HERE, "oracle.h")]

BC = {"periodic": 0, "transmissive": 1, "reflective": 2}
SCHEME = {"central4": 0, "weno5": 1}


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-O2 -ffp-contract=off, no fast-math)."""
    stale = not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in _SRC)
    if force or stale:
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-fopenmp",
               "-o", _SO + ".tmp", _SRC[0]]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Cfg(C.Structure):
    _fields_ = [("lo", C.c_double * 2), ("hi", C.c_double * 2), ("base", C.c_int * 2), ("n", C.c_int),
                ("levels", C.c_int), ("gamma", C.c_double), ("bc", C.c_int * 4), ("scheme", C.c_int),
                ("characteristic", C.c_int), ("div_order", C.c_int), ("weno_eps", C.c_double),
                ("theta", C.c_double), ("coarsen_frac", C.c_double), ("coarsen_rule", C.c_int),
                ("check_positivity", C.c_int), ("reflux", C.c_int)]


_lib = None
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_U8 = C.POINTER(C.c_uint8)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(_Cfg)]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_error.restype = C.c_char_p
        L.orc_error.argtypes = [C.c_void_p]
        L.orc_num_patches.argtypes = [C.c_void_p]
        L.orc_get_tree.argtypes = [C.c_void_p, C.c_int, _I, _I, _I, _I, _I]
        L.orc_validate.argtypes = [C.c_void_p]
        L.orc_set_patch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _D]
        L.orc_get_patch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _D]
        L.orc_restrict_all.argtypes = [C.c_void_p]
        L.orc_lambda.argtypes = [C.c_void_p, _D]
        L.orc_lambda_subcycled.argtypes = [C.c_void_p, _D]
        L.orc_stage1.argtypes = [C.c_void_p, C.c_double]
        L.orc_set_num_threads.argtypes = [C.c_int]
        L.orc_get_max_threads.restype = C.c_int
        L.orc_totals.argtypes = [C.c_void_p, _D]
        L.orc_step.argtypes = [C.c_void_p, C.c_double, C.c_double, _D]
        L.orc_step_subcycled.argtypes = [C.c_void_p, C.c_double, C.c_double, _D]
        L.orc_flags.argtypes = [C.c_void_p, C.c_int, _D, _U8, _U8, _U8]
        L.orc_regrid_with_requests.argtypes = [C.c_void_p, C.c_int, _I, _I, _I, _U8, _U8, _I, _I]
        L.orc_regrid.argtypes = [C.c_void_p, _I, _I]
        L.orc_ghost_tile.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _D]
        L.orc_rhs.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _D]
        L.orc_cons2prim.argtypes = [C.c_double, _D, _D]
        L.orc_prim2cons.argtypes = [C.c_double, _D, _D]
        L.orc_euler_flux_x.argtypes = [C.c_double, _D, _D]
        L.orc_rusanov_x.argtypes = [C.c_double, _D, _D, _D]
        L.orc_weno5.restype = C.c_double
        L.orc_weno5.argtypes = [_D, C.c_double]
        L.orc_eigen_x.argtypes = [C.c_double, _D, _D, _D, _D]
        L.orc_face_flux_x.argtypes = [C.POINTER(_Cfg), _D, _D]
        L.orc_mc.restype = C.c_double
        L.orc_mc.argtypes = [C.c_double, C.c_double]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def make_cfg(cfg: dict) -> _Cfg:
    """Marshal a workload dict (see workloads.py) into the oracle's own config struct."""
    c = _Cfg()
    c.lo[0], c.lo[1] = cfg["lo"]
    c.hi[0], c.hi[1] = cfg["hi"]
    c.base[0], c.base[1] = cfg["base"]
    c.n = cfg["n"]
    c.levels = cfg["levels"]
    c.gamma = cfg.get("gamma", 1.4)
    for e, b in enumerate(cfg["bc"]):
        c.bc[e] = BC[b]
    c.scheme = SCHEME[cfg["scheme"]]
    c.characteristic = int(cfg.get("characteristic", 1))
    c.div_order = int(cfg.get("div_order", 4))
    c.weno_eps = cfg.get("weno_eps", 1e-6)
    c.theta = cfg.get("theta", 0.1)
    c.coarsen_frac = cfg.get("coarsen_frac", 0.25)
    c.coarsen_rule = {"r2_exact": 0, "alg2_literal": 1}[cfg.get("coarsen_rule", "r2_exact")]
    c.check_positivity = int(cfg.get("check_positivity", 1))
    c.reflux = int(cfg.get("oracle_reflux", 1))   # test-only no-reflux control (oracle side only)
    return c


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class Oracle:
    """One composite AMR mesh advanced by the plain CPU definition (O1-O18)."""

    def __init__(self, cfg: dict):
        self.cfg = dict(cfg)
        self._c = make_cfg(cfg)
        self.h = lib().orc_create(C.byref(self._c))
        if not self.h:
            raise ValueError("oracle rejected config")
        self.n = cfg["n"]

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, lib().orc_error(self.h).decode())

    def tree(self):
        """Active patches in canonical (level, Q, P) order: list of (l, P, Q, leaf)."""
        m = lib().orc_num_patches(self.h)
        l, P, Q, lf, cl = (np.zeros(m, np.int32) for _ in range(5))
        self._chk(lib().orc_get_tree(self.h, m, *(a.ctypes.data_as(_I) for a in (l, P, Q, lf, cl))))
        return [(int(a), int(b), int(c), bool(d)) for a, b, c, d in zip(l, P, Q, lf)]

    def leaves(self):
        return [(l, P, Q) for (l, P, Q, lf) in self.tree() if lf]

    def validate(self):
        self._chk(lib().orc_validate(self.h))

    def set_patch(self, key, U):
        U = _f64(U)
        assert U.shape == (4, self.n, self.n)
        self._chk(lib().orc_set_patch(self.h, *key, _dp(U)))

    def get_patch(self, key):
        U = np.empty((4, self.n, self.n))
        self._chk(lib().orc_get_patch(self.h, *key, _dp(U)))
        return U

    def set_state(self, fn):
        """fn(l, P, Q) -> U[4][n][n] for every active patch, then restrict (O9)."""
        for (l, P, Q, _) in self.tree():
            self.set_patch((l, P, Q), fn(l, P, Q))
        self._chk(lib().orc_restrict_all(self.h))

    def get_state(self):
        return {(l, P, Q): self.get_patch((l, P, Q)) for (l, P, Q, _) in self.tree()}

    def restrict(self):
        self._chk(lib().orc_restrict_all(self.h))

    def lam(self):
        v = C.c_double()
        self._chk(lib().orc_lambda(self.h, C.byref(v)))
        return v.value

    def lam_subcycled(self):
        v = C.c_double()
        self._chk(lib().orc_lambda_subcycled(self.h, C.byref(v)))
        return v.value

    def stage1(self, dt):
        """O11 stage 1 alone (forward Euler with reflux and restriction) -- for the reflux-placement pin."""
        self._chk(lib().orc_stage1(self.h, float(dt)))

    def totals(self):
        out = np.zeros(4)
        self._chk(lib().orc_totals(self.h, _dp(out)))
        return out

    def step(self, dt=0.0, cfl=0.0, subcycle=False):
        """One step (O11); subcycle=True: one level-0 step with Berger-Colella time subcycling (NEXT #4)."""
        d = C.c_double()
        f = lib().orc_step_subcycled if subcycle else lib().orc_step
        self._chk(f(self.h, float(dt), float(cfl), C.byref(d)))
        return d.value

    def flags(self):
        """Per active patch (canonical order): dict key -> (maxeta, refine, coarsen, ambiguous)."""
        tr = self.tree()
        m = len(tr)
        me = np.zeros(m)
        rf, cf, am = (np.zeros(m, np.uint8) for _ in range(3))
        self._chk(lib().orc_flags(self.h, m, _dp(me), *(a.ctypes.data_as(_U8) for a in (rf, cf, am))))
        return {(l, P, Q): (float(me[e]), bool(rf[e]), bool(cf[e]), bool(am[e]))
                for e, (l, P, Q, _) in enumerate(tr)}

    def regrid_with_requests(self, refine_keys=(), coarsen_keys=()):
        keys = sorted(set(refine_keys) | set(coarsen_keys))
        m = len(keys)
        l = np.array([k[0] for k in keys], np.int32)
        P = np.array([k[1] for k in keys], np.int32)
        Q = np.array([k[2] for k in keys], np.int32)
        rs, cs = set(refine_keys), set(coarsen_keys)
        rf = np.array([k in rs for k in keys], np.uint8)
        cf = np.array([k in cs for k in keys], np.uint8)
        nr, nc = C.c_int(), C.c_int()
        self._chk(lib().orc_regrid_with_requests(self.h, m, *(a.ctypes.data_as(_I) for a in (l, P, Q)),
                                                 rf.ctypes.data_as(_U8), cf.ctypes.data_as(_U8),
                                                 C.byref(nr), C.byref(nc)))
        return nr.value, nc.value

    def regrid(self):
        nr, nc = C.c_int(), C.c_int()
        self._chk(lib().orc_regrid(self.h, C.byref(nr), C.byref(nc)))
        return nr.value, nc.value

    def ghost_tile(self, key, g):
        w = self.n + 2 * g
        t = np.empty((4, w, w))
        self._chk(lib().orc_ghost_tile(self.h, *key, g, _dp(t)))
        return t

    def rhs(self, key):
        L = np.empty((4, self.n, self.n))
        self._chk(lib().orc_rhs(self.h, *key, _dp(L)))
        return L


# ---- unit-level functions (pins) ----
def cons2prim(U, gamma=1.4):
    U = _f64(U); W = np.empty(4); lib().orc_cons2prim(gamma, _dp(U), _dp(W)); return W


def prim2cons(W, gamma=1.4):
    W = _f64(W); U = np.empty(4); lib().orc_prim2cons(gamma, _dp(W), _dp(U)); return U


def euler_flux_x(U, gamma=1.4):
    U = _f64(U); F = np.empty(4); lib().orc_euler_flux_x(gamma, _dp(U), _dp(F)); return F


def rusanov_x(UL, UR, gamma=1.4):
    UL, UR = _f64(UL), _f64(UR); F = np.empty(4); lib().orc_rusanov_x(gamma, _dp(UL), _dp(UR), _dp(F)); return F


def weno5(v, eps=1e-6):
    v = _f64(v); return lib().orc_weno5(_dp(v), eps)


def eigen_x(WL, WR, gamma=1.4):
    WL, WR = _f64(WL), _f64(WR)
    Lm, Rm = np.empty(16), np.empty(16)
    lib().orc_eigen_x(gamma, _dp(WL), _dp(WR), _dp(Lm), _dp(Rm))
    return Lm.reshape(4, 4), Rm.reshape(4, 4)


def face_flux_x(cfg: dict, cells):
    c = make_cfg(cfg); cells = _f64(cells); assert cells.shape == (6, 4)
    F = np.empty(4); lib().orc_face_flux_x(C.byref(c), _dp(cells), _dp(F)); return F


def set_num_threads(n: int):
    """OpenMP threads of the oracle (over patches; results do not depend on it)."""
    lib().orc_set_num_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_get_max_threads())


def mc(a, b):
    return lib().orc_mc(a, b)
