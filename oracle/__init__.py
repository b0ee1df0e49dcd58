"""Parity oracle for arXiv 1502.01629's hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package.  The product path
(``paper_1502_01629_b200``) never imports it and shares no code with it; both consume the
arrays built by ``pdd_inputs``.

This module is the thin ctypes marshalling layer over ``pdd_oracle.c`` (plain fp64 C with
OpenMP over rows; see that file's header for the passage each function follows) plus
``solve_pipeline`` which strings the paper's steps together in the order of P:811-843.

Parity status of each function:
  node update / Jacobi fixed point : pinned (P1-P14 in tests/test_oracle_pins.py)
  prolongation                     : pinned (P16)
  synthesis                        : pinned (P17)
  successor labels                 : rule is a convention (R17/R18); pinned only by invariants
                                     (label constant along chains, chain reaches its sector,
                                     N_P = 1) -- "parity unpinned" beyond those.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pdd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
          "-std=c11", "-Wall"]


def build(force: bool = False) -> str:
    """Compile oracle/pdd_oracle.c -> oracle/liboracle.so (gcc, fp-contract off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


class _Coef(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value", C.c_double), ("data", C.POINTER(C.c_double))]


class _Problem(C.Structure):
    _fields_ = [("n", C.c_int32), ("lo", C.c_double), ("dx", C.c_double), ("h", C.c_double),
                ("lam", C.c_double), ("na", C.c_int32), ("ctrl", C.POINTER(C.c_double)),
                ("speed", _Coef), ("drift", _Coef * 2), ("p", C.c_int32),
                ("sigma", (_Coef * 2) * 2), ("cost", _Coef), ("diffusion_scale", C.c_int32),
                ("kind", C.POINTER(C.c_uint8)), ("sigma_mode", C.c_int32),
                ("cost_ctrl", C.POINTER(C.c_double))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int64)
        P = C.POINTER(_Problem)
        L.orc_num_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_beta.argtypes = [P]
        L.orc_beta.restype = C.c_double
        L.orc_init_v0.argtypes = [P, dp]
        L.orc_bilinear_weights.argtypes = [C.c_int, C.c_double, C.c_double, ip, dp]
        L.orc_node_update.argtypes = [P, dp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int32)]
        L.orc_node_update.restype = C.c_double
        L.orc_node_lambdas.argtypes = [P, dp, C.c_int, C.c_int, dp, dp]
        L.orc_apply.argtypes = [P, dp, dp, C.c_int, C.POINTER(C.c_int32)]
        L.orc_apply.restype = C.c_double
        L.orc_apply_at.argtypes = [P, dp, ip, C.c_int64, dp, C.POINTER(C.c_int32)]
        L.orc_jacobi.argtypes = [P, dp, C.c_double, C.c_int64, C.c_int, dp, dp]
        L.orc_jacobi.restype = C.c_int64
        L.orc_gauss_seidel.argtypes = [P, dp, ip, C.c_int64, C.c_double, C.c_int64, C.c_int, dp]
        L.orc_gauss_seidel.restype = C.c_int64
        L.orc_prolong.argtypes = [C.c_int, dp, C.c_int, dp]
        L.orc_prolong.restype = C.c_int
        L.orc_synthesize.argtypes = [P, dp, C.POINTER(C.c_uint8)]
        L.orc_successor.argtypes = [P, C.POINTER(C.c_uint8), C.c_double, ip]
        L.orc_labels.argtypes = [P, ip, C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_int16)]
        L.orc_labels.restype = C.c_int
        L.orc_label_at.argtypes = [P, C.c_int, dp, C.POINTER(C.c_int32), C.c_int, C.c_double,
                                   C.c_int64, C.c_int64]
        L.orc_label_at.restype = C.c_int32
        L.orc_astar_at.argtypes = [P, C.c_int, dp, ip, C.c_int64, C.POINTER(C.c_int32)]
        L.orc_uhat_at.argtypes = [C.c_int, C.c_int, dp, ip, C.c_int64, dp]
        L.orc_static_labels.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8),
                                        C.POINTER(C.c_int16)]
        L.orc_fuzzy_phi.argtypes = [P, C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.c_int,
                                    C.c_double, C.c_int64, dp, dp]
        L.orc_fuzzy_phi.restype = C.c_int64
        L.orc_fuzzy_sparse.argtypes = [P, C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.c_int, C.c_int,
                                       C.c_double, C.c_int64, C.POINTER(C.c_int16), dp, dp]
        L.orc_fuzzy_sparse.restype = C.c_int64
        L.orc_fuzzy_sparse_assign.argtypes = [P, C.POINTER(C.c_int16), dp, C.c_int, C.c_int, C.c_double,
                                              C.POINTER(C.c_int16), C.POINTER(C.c_uint8)]
        L.orc_fuzzy_assign.argtypes = [P, dp, C.c_int, C.c_double, C.POINTER(C.c_int16),
                                       C.POINTER(C.c_uint8)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Problem:
    """ctypes view of a ``pdd_inputs.Instance`` (keeps the arrays alive)."""

    def __init__(self, inst):
        self.inst = inst
        self._keep = []
        s = _Problem()
        s.n, s.lo, s.dx, s.h, s.lam = inst.n, inst.lo, inst.dx, inst.h, inst.lam
        ctrl = np.ascontiguousarray(inst.controls, dtype=np.float64).reshape(-1)
        self._keep.append(ctrl)
        s.na, s.ctrl = inst.n_controls, _ptr(ctrl, C.c_double)
        s.speed = self._coef(inst.speed)
        s.drift[0] = self._coef(inst.drift[0])
        s.drift[1] = self._coef(inst.drift[1])
        s.p = inst.p
        for k in range(2):
            for c in range(2):
                s.sigma[k][c] = self._coef(inst.sigma[k][c])
        s.cost = self._coef(inst.cost)
        s.diffusion_scale = inst.diffusion_scale
        kind = np.ascontiguousarray(inst.kind, dtype=np.uint8)
        self._keep.append(kind)
        s.kind = _ptr(kind, C.c_uint8)
        s.sigma_mode = int(getattr(inst, "sigma_mode", 0))
        cc = getattr(inst, "cost_ctrl", None)
        if cc is not None:
            cc = np.ascontiguousarray(cc, dtype=np.float64)
            self._keep.append(cc)
            s.cost_ctrl = _ptr(cc, C.c_double)
        self.s = s

    def _coef(self, c):
        out = _Coef()
        out.kind, out.value = c.kind, c.value
        if c.data is not None:
            d = np.ascontiguousarray(c.data, dtype=np.float64)
            self._keep.append(d)
            out.data = _ptr(d, C.c_double)
        return out

    @property
    def ref(self):
        return C.byref(self.s)


# ------------------------------------------------------------------------------------------
# thin wrappers
# ------------------------------------------------------------------------------------------

def num_threads() -> int:
    return lib().orc_num_threads()


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def beta(inst) -> float:
    return lib().orc_beta(Problem(inst).ref)


def init_v0(inst) -> np.ndarray:
    P = Problem(inst)
    V = np.empty(inst.n * inst.n, dtype=np.float64)
    lib().orc_init_v0(P.ref, _ptr(V, C.c_double))
    return V


def bilinear_weights(n: int, gx: float, gy: float):
    cr = np.zeros(4, dtype=np.int64)
    w = np.zeros(4, dtype=np.float64)
    lib().orc_bilinear_weights(n, gx, gy, _ptr(cr, C.c_int64), _ptr(w, C.c_double))
    return cr, w


def node_update(inst, V: np.ndarray, i: int, j: int, scheme: int = 0):
    P = Problem(inst)
    V = np.ascontiguousarray(V, dtype=np.float64)
    a = C.c_int32(-1)
    v = lib().orc_node_update(P.ref, _ptr(V, C.c_double), i, j, scheme, C.byref(a))
    return v, a.value


def node_lambdas(inst, V: np.ndarray, i: int, j: int):
    P = Problem(inst)
    V = np.ascontiguousarray(V, dtype=np.float64)
    l0 = np.zeros(inst.n_controls)
    rp = np.zeros(inst.n_controls)
    lib().orc_node_lambdas(P.ref, _ptr(V, C.c_double), i, j, _ptr(l0, C.c_double),
                           _ptr(rp, C.c_double))
    return l0, rp


def apply(inst, V: np.ndarray, scheme: int = 0, with_argmin: bool = False):
    P = Problem(inst)
    V = np.ascontiguousarray(V, dtype=np.float64)
    out = np.empty_like(V)
    am = np.empty(V.size, dtype=np.int32) if with_argmin else None
    res = lib().orc_apply(P.ref, _ptr(V, C.c_double), _ptr(out, C.c_double), scheme,
                          _ptr(am, C.c_int32) if am is not None else None)
    return (out, res, am) if with_argmin else (out, res)


def apply_at(inst, V: np.ndarray, idx: np.ndarray):
    P = Problem(inst)
    V = np.ascontiguousarray(V, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.size, dtype=np.float64)
    am = np.empty(idx.size, dtype=np.int32)
    lib().orc_apply_at(P.ref, _ptr(V, C.c_double), _ptr(idx, C.c_int64), idx.size,
                       _ptr(out, C.c_double), _ptr(am, C.c_int32))
    return out, am


def jacobi(inst, V0: Optional[np.ndarray] = None, tol: float = 1e-9, max_sweeps: int = 10**7,
           scheme: int = 0, history: bool = False):
    """Jacobi value iteration from V0 (default: the constant supersolution, R11)."""
    P = Problem(inst)
    V = init_v0(inst) if V0 is None else np.array(V0, dtype=np.float64, copy=True)
    res = C.c_double(0.0)
    hist = np.zeros(int(min(max_sweeps, 10**6)), dtype=np.float64) if history else None
    s = lib().orc_jacobi(P.ref, _ptr(V, C.c_double), tol, max_sweeps, scheme, C.byref(res),
                         _ptr(hist, C.c_double) if hist is not None else None)
    out = dict(V=V, sweeps=int(s), residual=res.value)
    if history:
        out["history"] = hist[:s]
    return out


def gauss_seidel(inst, order: np.ndarray, V0: Optional[np.ndarray] = None, tol: float = 1e-9,
                 max_sweeps: int = 10**6, scheme: int = 0):
    P = Problem(inst)
    V = init_v0(inst) if V0 is None else np.array(V0, dtype=np.float64, copy=True)
    order = np.ascontiguousarray(order, dtype=np.int64)
    res = C.c_double(0.0)
    s = lib().orc_gauss_seidel(P.ref, _ptr(V, C.c_double), _ptr(order, C.c_int64), order.size,
                               tol, max_sweeps, scheme, C.byref(res))
    return dict(V=V, sweeps=int(s), residual=res.value)


def prolong(nc: int, uc: np.ndarray, n: int) -> np.ndarray:
    uc = np.ascontiguousarray(uc, dtype=np.float64)
    out = np.empty(n * n, dtype=np.float64)
    if lib().orc_prolong(nc, _ptr(uc, C.c_double), n, _ptr(out, C.c_double)) != 0:
        raise ValueError("coarse grid does not nest in the fine grid")
    return out


def synthesize(inst, uhat: np.ndarray) -> np.ndarray:
    P = Problem(inst)
    uhat = np.ascontiguousarray(uhat, dtype=np.float64)
    out = np.empty(inst.n * inst.n, dtype=np.uint8)
    lib().orc_synthesize(P.ref, _ptr(uhat, C.c_double), _ptr(out, C.c_uint8))
    return out


SUCCESSOR_M = 4.0   # R18: jump length in cells


def successor(inst, astar: np.ndarray, M: float = SUCCESSOR_M) -> np.ndarray:
    P = Problem(inst)
    astar = np.ascontiguousarray(astar, dtype=np.uint8)
    out = np.empty(inst.n * inst.n, dtype=np.int64)
    lib().orc_successor(P.ref, _ptr(astar, C.c_uint8), M, _ptr(out, C.c_int64))
    return out


def labels(inst, succ: np.ndarray, n_patches: Optional[int] = None) -> np.ndarray:
    P = Problem(inst)
    succ = np.ascontiguousarray(succ, dtype=np.int64)
    sec = np.ascontiguousarray(inst.sector, dtype=np.int32)
    out = np.empty(inst.n * inst.n, dtype=np.int16)
    npch = inst.n_patches if n_patches is None else n_patches
    if lib().orc_labels(P.ref, _ptr(succ, C.c_int64), _ptr(sec, C.c_int32), npch,
                        _ptr(out, C.c_int16)) != 0:
        raise MemoryError
    return out


def label_at(inst, uc: np.ndarray, k: int, M: float = SUCCESSOR_M) -> int:
    P = Problem(inst)
    uc = np.ascontiguousarray(uc, dtype=np.float64)
    sec = np.ascontiguousarray(inst.sector, dtype=np.int32)
    return int(lib().orc_label_at(P.ref, inst.coarse.n, _ptr(uc, C.c_double),
                                  _ptr(sec, C.c_int32), inst.n_patches, M, int(k),
                                  inst.n * inst.n + 1))


def astar_at(inst, uc: np.ndarray, idx: np.ndarray) -> np.ndarray:
    P = Problem(inst)
    uc = np.ascontiguousarray(uc, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.size, dtype=np.int32)
    lib().orc_astar_at(P.ref, inst.coarse.n, _ptr(uc, C.c_double), _ptr(idx, C.c_int64),
                       idx.size, _ptr(out, C.c_int32))
    return out


def uhat_at(inst, uc: np.ndarray, idx: np.ndarray) -> np.ndarray:
    uc = np.ascontiguousarray(uc, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.size, dtype=np.float64)
    lib().orc_uhat_at(inst.n, inst.coarse.n, _ptr(uc, C.c_double), _ptr(idx, C.c_int64),
                      idx.size, _ptr(out, C.c_double))
    return out


def static_labels(inst, px: Optional[int] = None, py: Optional[int] = None) -> np.ndarray:
    px = inst.static_blocks[0] if px is None else px
    py = inst.static_blocks[1] if py is None else py
    kind = np.ascontiguousarray(inst.kind, dtype=np.uint8)
    out = np.empty(inst.n * inst.n, dtype=np.int16)
    lib().orc_static_labels(inst.n, px, py, _ptr(kind, C.c_uint8), _ptr(out, C.c_int16))
    return out


# ------------------------------------------------------------------------------------------
# the paper's pipeline, plain and sequential
# ------------------------------------------------------------------------------------------

def coarse_solve(inst, tol_c: Optional[float] = None, max_sweeps: int = 10**6):
    """u_c: SL fixed point with sigma = 0 on G_c from V0, until residual < eps_c."""
    c = inst.coarse
    return jacobi(c, tol=inst.tol_coarse if tol_c is None else tol_c, max_sweeps=max_sweeps)


def solve_pipeline(inst, tol: Optional[float] = None, fine: bool = True,
                   max_sweeps: int = 10**7):
    """Pre-computation (coarse solve, prolongation, synthesis, successor labels, static labels)
    and the fine-grid fixed point by Jacobi from V0.  Returns a dict with timings."""
    out = {}
    t0 = time.perf_counter()
    if inst.coarse is not None:
        cs = coarse_solve(inst)
        out["uc"], out["coarse_sweeps"], out["coarse_residual"] = cs["V"], cs["sweeps"], cs["residual"]
        out["uhat"] = prolong(inst.coarse.n, cs["V"], inst.n)
        out["astar"] = synthesize(inst, out["uhat"])
        out["succ"] = successor(inst, out["astar"])
        out["labels"] = labels(inst, out["succ"])
    out["static_labels"] = static_labels(inst)
    out["seconds_precompute"] = time.perf_counter() - t0
    if fine:
        t1 = time.perf_counter()
        fs = jacobi(inst, tol=inst.tol if tol is None else tol, max_sweeps=max_sweeps)
        out["seconds_fine"] = time.perf_counter() - t1
        out["V"], out["sweeps"], out["residual"] = fs["V"], fs["sweeps"], fs["residual"]
    out["threads"] = num_threads()
    return out


def fuzzy_phi(inst, astar: np.ndarray, n_patches: int, eps_P: float, max_sweeps: int = 10**6):
    """phi_p of the paper's fuzzy patches: Jacobi of the SL advection scheme along the
    synthesised field until the sweep change is < eps_P.  Returns dict(phi (n_patches, N),
    sweeps, residual)."""
    P = Problem(inst)
    N = inst.n * inst.n
    a = np.ascontiguousarray(astar, dtype=np.uint8)
    sec = np.ascontiguousarray(inst.sector, dtype=np.int32)
    phi = np.empty(n_patches * N, dtype=np.float64)
    res = C.c_double(0.0)
    sw = lib().orc_fuzzy_phi(P.ref, _ptr(a, C.c_uint8), _ptr(sec, C.c_int32), int(n_patches),
                             float(eps_P), int(max_sweeps), _ptr(phi, C.c_double), C.byref(res))
    return {"phi": phi.reshape(n_patches, N), "sweeps": int(sw), "residual": res.value}


def fuzzy_assign(inst, phi: np.ndarray, tau_P: float):
    """Thresholding / ownership of the fuzzy patches (R38): (labels, members)."""
    P = Problem(inst)
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    npatch = phi.shape[0]
    N = inst.n * inst.n
    lab = np.empty(N, dtype=np.int16)
    mem = np.empty(N, dtype=np.uint8)
    lib().orc_fuzzy_assign(P.ref, _ptr(phi.reshape(-1), C.c_double), int(npatch), float(tau_P),
                           _ptr(lab, C.c_int16), _ptr(mem, C.c_uint8))
    return lab, mem


def fuzzy_sparse(inst, astar: np.ndarray, n_patches: int, K: int, eps_P: float, tau_P: float = 0.5,
                 max_sweeps: int = 10**6):
    """Sparse top-K form of the fuzzy patches (per node the K largest (patch, phi_p) pairs; reading
    R40).  Returns dict(lab (N, K) int16, mass (N, K), sweeps, residual, labels, members)."""
    P = Problem(inst)
    N = inst.n * inst.n
    a = np.ascontiguousarray(astar, dtype=np.uint8)
    sec = np.ascontiguousarray(inst.sector, dtype=np.int32)
    lab = np.empty(N * K, dtype=np.int16)
    mass = np.empty(N * K, dtype=np.float64)
    res = C.c_double(0.0)
    sw = lib().orc_fuzzy_sparse(P.ref, _ptr(a, C.c_uint8), _ptr(sec, C.c_int32), int(n_patches), int(K),
                                float(eps_P), int(max_sweeps), _ptr(lab, C.c_int16),
                                _ptr(mass, C.c_double), C.byref(res))
    if sw < 0:
        raise ValueError("K must be in 1..16")
    own = np.empty(N, dtype=np.int16)
    mem = np.empty(N, dtype=np.uint8)
    lib().orc_fuzzy_sparse_assign(P.ref, _ptr(lab, C.c_int16), _ptr(mass, C.c_double), int(K),
                                  int(n_patches), float(tau_P), _ptr(own, C.c_int16), _ptr(mem, C.c_uint8))
    return {"lab": lab.reshape(N, K), "mass": mass.reshape(N, K), "sweeps": int(sw),
            "residual": res.value, "labels": own, "members": mem}
