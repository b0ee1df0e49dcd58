"""paper_1502_01629_b200 -- B200-native hot path of the patchy domain decomposition method for
stationary second-order HJB equations (arXiv 1502.01629).

The compute lives in ``libpdd.so`` (hand-written sm_100a CUDA + a C++ host runtime behind the C
ABI of ``include/pdd.h``).  This module is the thin Python binding with the same call names:
argument marshalling only.  PyTorch provides the device workspace and the CUDA stream.

Problem objects are duck-typed: anything with the attributes of ``pdd_inputs.Instance``
(n, lo, hi, dx, h, lam, controls, speed, drift, p, sigma, cost, diffusion_scale, kind, sector,
coarse) works.  Coefficients expose ``kind`` (0 const, 1 row, 2 col, 3 field), ``value``, ``data``.

Typical use (the paper's algorithm)::

    s = Solver(instance, precision=32)
    s.coarse_solve(1e-12)            # u_c on G_c
    s.synthesize()                   # u_hat, a*
    s.build_patches(instance.n_patches)
    st = s.solve(mode="patchy", tol=1e-6)
    V = s.get_values()
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _native as N

__all__ = ["Solver", "PddError", "version", "MODE_PATCHY", "MODE_STATIC"]

MODE_PATCHY, MODE_STATIC = 0, 1


class PddError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{N.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def version() -> str:
    return N.lib().pdd_version().decode()


def _check(st: int, ctx=None):
    if st != N.PDD_OK:
        msg = N.lib().pdd_last_error(ctx)
        raise PddError(st, msg.decode() if msg else "")


class _ProblemView:
    """ctypes ``pdd_problem`` built from a duck-typed instance; keeps host arrays alive."""

    def __init__(self, inst, with_sector: bool = True, pin: bool = False):
        self._keep = []
        s = N.pdd_problem()
        s.n = int(inst.n)
        s.lo, s.hi, s.dx, s.h, s.lam = (float(inst.lo), float(inst.hi), float(inst.dx),
                                         float(inst.h), float(inst.lam))
        ctrl = self._arr(np.asarray(inst.controls, dtype=np.float64).reshape(-1), pin)
        s.n_controls = int(np.asarray(inst.controls).shape[0])
        s.controls = ctrl.ctypes.data_as(C.POINTER(C.c_double))
        s.speed = self._coef(inst.speed, pin)
        s.drift[0] = self._coef(inst.drift[0], pin)
        s.drift[1] = self._coef(inst.drift[1], pin)
        s.p = int(inst.p)
        for k in range(2):
            for c in range(2):
                s.sigma[k][c] = self._coef(inst.sigma[k][c], pin)
        s.cost = self._coef(inst.cost, pin)
        s.diffusion_scale = int(getattr(inst, "diffusion_scale", 0))
        kind = self._arr(np.asarray(inst.kind, dtype=np.uint8).reshape(-1), pin)
        s.kind = kind.ctypes.data_as(C.POINTER(C.c_uint8))
        sector = getattr(inst, "sector", None)
        if with_sector and sector is not None:
            sec = self._arr(np.asarray(sector).astype(np.int16).reshape(-1), pin)
            s.sector = sec.ctypes.data_as(C.POINTER(C.c_int16))
        s.sigma_mode = int(getattr(inst, "sigma_mode", 0))
        cc = getattr(inst, "cost_ctrl", None)
        if cc is not None:
            cca = self._arr(np.asarray(cc, dtype=np.float64).reshape(-1), pin)
            s.cost_ctrl = cca.ctypes.data_as(C.POINTER(C.c_double))
        self.s = s

    def _arr(self, a: np.ndarray, pin: bool):
        a = np.ascontiguousarray(a)
        if pin and a.nbytes >= (1 << 16):
            import torch
            t = torch.from_numpy(a.copy()).pin_memory()
            self._keep.append(t)
            a = t.numpy()
        self._keep.append(a)
        return a

    def _coef(self, c, pin):
        out = N.pdd_coef()
        out.kind, out.value = int(c.kind), float(c.value)
        if c.data is not None and int(c.kind) != 0:
            d = self._arr(np.asarray(c.data, dtype=np.float64).reshape(-1), pin)
            out.data = d.ctypes.data_as(C.POINTER(C.c_double))
        return out


class Solver:
    """One problem instance on one GPU: wraps a ``pdd_ctx``."""

    def __init__(self, inst, precision: int = 32, device: str = "cuda", stream=None,
                 pin_host: bool = False, views=None):
        import torch
        self.inst = inst
        self.n = int(inst.n)
        self.precision = int(precision)
        self.device = torch.device(device)
        L = N.lib()
        if views is None:
            views = (_ProblemView(inst, True, pin_host),
                     _ProblemView(inst.coarse, False, pin_host) if getattr(inst, "coarse", None) is not None else None)
        self._fine, self._coarse = views
        fp = C.byref(self._fine.s)
        cp = C.byref(self._coarse.s) if self._coarse is not None else None
        nbytes = C.c_size_t(0)
        _check(L.pdd_workspace_bytes(fp, cp, self.precision, C.byref(nbytes)))
        self.workspace = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device=self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._ctx = C.c_void_p()
        _check(L.pdd_create(fp, cp, self.precision, C.c_void_p(self.stream.cuda_stream),
                            C.c_void_p(self.workspace.data_ptr()), int(nbytes.value) + 256,
                            C.byref(self._ctx)))

    @staticmethod
    def make_views(inst, pin_host: bool = True):
        """Host-side marshalled (optionally pinned) copies of an instance, reusable across
        Solver constructions (the e2e bench builds them once, outside its timed region)."""
        return (_ProblemView(inst, True, pin_host),
                _ProblemView(inst.coarse, False, pin_host) if getattr(inst, "coarse", None) is not None else None)

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            N.lib().pdd_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, st):
        _check(st, self._ctx)

    # ------------------------------------------------------------------ the method
    def coarse_solve(self, tol_c: float = 1e-12, max_sweeps: int = 1 << 20) -> dict:
        st = N.pdd_coarse_stats()
        self._ck(N.lib().pdd_coarse_solve(self._ctx, tol_c, max_sweeps, C.byref(st)))
        return st.as_dict()

    def synthesize(self) -> None:
        self._ck(N.lib().pdd_synthesize(self._ctx))

    def build_patches(self, n_patches: int, M: float = 4.0) -> None:
        self._ck(N.lib().pdd_build_patches(self._ctx, int(n_patches), float(M)))

    def build_fuzzy_patches(self, n_patches: int, eps_P: float = 1e-3, tau_P: float = 0.5,
                            max_sweeps: int = 1 << 20, return_phi: bool = False) -> dict:
        """The paper's fuzzy patches: phi_p advected along the feedback until the
        sweep change is < eps_P, thresholded at tau_P (owner = largest phi_p).  The device
        scratch (two n_patches x n^2 fp64 fields) is a torch tensor owned here."""
        import torch
        nb = C.c_size_t(0)
        _check(N.lib().pdd_fuzzy_scratch_bytes(int(self.n), int(n_patches), C.byref(nb)), None)
        scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
        st = N.pdd_fuzzy_stats()
        self._ck(N.lib().pdd_build_fuzzy_patches(self._ctx, int(n_patches), float(eps_P),
                                                 float(tau_P), int(max_sweeps),
                                                 C.c_void_p(scratch.data_ptr()), int(nb.value),
                                                 C.byref(st)))
        out = st.as_dict()
        if return_phi:
            nn = self.n * self.n
            off = int(st.phi_offset)
            out["phi"] = scratch[off:off + 8 * nn * int(n_patches)].view(torch.float64) \
                .reshape(int(n_patches), nn).cpu().numpy()
        del scratch
        return out

    def build_fuzzy_patches_sparse(self, n_patches: int, K: int = 4, eps_P: float = 1e-3,
                                   tau_P: float = 0.5, max_sweeps: int = 1 << 20,
                                   return_lists: bool = False) -> dict:
        """Fuzzy patches in sparse form: per node the K largest (patch, phi_p) pairs (hundreds of
        patches; 20 K n^2 bytes of device scratch, a torch tensor owned here)."""
        import torch
        nb = C.c_size_t(0)
        _check(N.lib().pdd_fuzzy_sparse_scratch_bytes(int(self.n), int(K), C.byref(nb)), None)
        scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
        st = N.pdd_fuzzy_stats()
        self._ck(N.lib().pdd_build_fuzzy_patches_sparse(self._ctx, int(n_patches), int(K), float(eps_P),
                                                        float(tau_P), int(max_sweeps),
                                                        C.c_void_p(scratch.data_ptr()), int(nb.value),
                                                        C.byref(st)))
        out = st.as_dict()
        if return_lists:
            nk = self.n * self.n * int(K)
            po, lo = int(st.phi_offset), int(st.lab_offset)
            out["mass"] = scratch[po:po + 8 * nk].view(torch.float64).reshape(-1, int(K)).cpu().numpy()
            out["lab"] = scratch[lo:lo + 2 * nk].view(torch.int16).reshape(-1, int(K)).cpu().numpy()
        del scratch
        return out

    def build_static(self, px: int, py: int) -> None:
        self._ck(N.lib().pdd_build_static(self._ctx, int(px), int(py)))

    def solve(self, mode="patchy", tol: float = 1e-6, k_inner: Optional[int] = None,
              max_rounds: int = 200000, delta: float = 0.0, kernel: int = 0,
              schedule: str = "auto", raise_on_noconverge: bool = True,
              early_exit: bool = True, bucket_policy: int = 0, trace: bool = False,
              queue_target: int = 0) -> dict:
        o = N.pdd_solve_opts()
        o.mode = MODE_PATCHY if mode in ("patchy", 0) else MODE_STATIC
        if k_inner is None:   # 0 = automatic in libpdd: 1 patchy / 4 static,
            k_inner = 0       # 4 for a patchy grid that fits one wave of sweep CTAs
        o.k_inner, o.tol, o.max_rounds, o.delta, o.kernel = int(k_inner), float(tol), int(max_rounds), float(delta), int(kernel)
        o.schedule = {"auto": 0, "ordered": 1, "queue": 2, "rounds": 3}.get(schedule, schedule)
        o.queue_target = int(queue_target)
        o.early_exit_off = 0 if early_exit else 1
        o.bucket_policy = int(bucket_policy)
        o.trace = 1 if trace else 0
        st = N.pdd_solve_stats()
        r = N.lib().pdd_solve(self._ctx, C.byref(o), C.byref(st))
        if r != N.PDD_OK and (raise_on_noconverge or r != N.PDD_E_NOCONVERGE):
            self._ck(r)
        return st.as_dict()

    def apply_operator(self, V: Optional[np.ndarray] = None, kernel: int = 0):
        """T(V) on every node (fp64 numpy array) and max |T(V) - V| over free nodes."""
        import torch
        if V is not None:
            self.set_values(V)
        out = torch.empty(self.n * self.n, dtype=torch.float64, device=self.device)
        res = C.c_double(0.0)
        self._ck(N.lib().pdd_apply_operator(self._ctx, C.c_void_p(out.data_ptr()), int(kernel),
                                            C.byref(res)))
        return out.cpu().numpy(), res.value

    # ------------------------------------------------------------------ fetch / set
    def _get(self, fn, dtype, count):
        a = np.empty(count, dtype=dtype)
        self._ck(fn(self._ctx, C.c_void_p(a.ctypes.data), 0))
        return a

    def get_values(self, as_fp64: bool = True) -> np.ndarray:
        a = np.empty(self.n * self.n, dtype=np.float64 if as_fp64 else np.float32)
        self._ck(N.lib().pdd_get_values(self._ctx, C.c_void_p(a.ctypes.data), 0, int(as_fp64)))
        return a

    def get_values_into(self, dst, on_device: bool, as_fp64: bool = True) -> None:
        """Copy V into a caller buffer (torch tensor or numpy array)."""
        ptr = dst.data_ptr() if hasattr(dst, "data_ptr") else dst.ctypes.data
        self._ck(N.lib().pdd_get_values(self._ctx, C.c_void_p(ptr), int(on_device), int(as_fp64)))

    def set_values(self, V: np.ndarray) -> None:
        V = np.ascontiguousarray(V, dtype=np.float64).reshape(-1)
        self._ck(N.lib().pdd_set_values(self._ctx, C.c_void_p(V.ctypes.data), 0))

    def get_uhat(self) -> np.ndarray:
        return self._get(N.lib().pdd_get_uhat, np.float64, self.n * self.n)

    def get_coarse_values(self) -> np.ndarray:
        nc = int(self.inst.coarse.n)
        return self._get(N.lib().pdd_get_coarse_values, np.float64, nc * nc)

    def get_controls(self) -> np.ndarray:
        return self._get(N.lib().pdd_get_controls, np.uint8, self.n * self.n)

    def get_labels(self) -> np.ndarray:
        return self._get(N.lib().pdd_get_labels, np.int16, self.n * self.n)

    def get_successors(self) -> np.ndarray:
        return self._get(N.lib().pdd_get_successors, np.int32, self.n * self.n)

    def get_patch_rounds(self, count: int) -> np.ndarray:
        a = np.empty(count, dtype=np.int32)
        self._ck(N.lib().pdd_get_patch_rounds(self._ctx, C.c_void_p(a.ctypes.data), int(count)))
        return a

    def get_patch_residuals(self, count: int) -> np.ndarray:
        a = np.empty(count, dtype=np.float64)
        self._ck(N.lib().pdd_get_patch_residuals(self._ctx, C.c_void_p(a.ctypes.data), int(count)))
        return a

    def get_tile_rounds(self, count: int) -> np.ndarray:
        a = np.empty(count, dtype=np.int32)
        self._ck(N.lib().pdd_get_tile_rounds(self._ctx, C.c_void_p(a.ctypes.data), int(count)))
        return a

    def set_tile_cols(self, cols: int) -> None:
        """Force the fp32 row-table tile geometry (0 auto, 64 or 128; A/B and tests)."""
        self._ck(N.lib().pdd_set_tile_cols(self._ctx, int(cols)))

    def set_tile_shape(self, rows: int, cols: int) -> None:
        """Force the fp32 row-table kernel's tile: (0, 0) automatic, (32, 64), (16, 128), (16, 64)."""
        self._ck(N.lib().pdd_set_tile_shape(self._ctx, int(rows), int(cols)))

    def kernel_launches(self) -> int:
        return int(N.lib().pdd_kernel_launches(self._ctx))

    # ------------------------------------------------------------------ convenience
    def run_patchy(self, tol: float, k_inner: Optional[int] = None, tol_c: float = 1e-12, **kw) -> dict:
        out = {"coarse": self.coarse_solve(tol_c)}
        self.synthesize()
        self.build_patches(self.inst.n_patches)
        out["fine"] = self.solve("patchy", tol=tol, k_inner=k_inner, **kw)
        return out


def regime_analyse(f_min: float, f_max: float, sigma_norm: float, dx: float) -> dict:
    """The upwind diffusion ball analysis of P:528-697 through the C ABI (pdd_regime_analyse):
    omega, upsilon, alpha bounds, the hyperbolicity flag, the paper's time step h = alpha dx /
    f_min and the eps threshold of sigma = sqrt(2 eps) I."""
    r = N.pdd_regime()
    st = N.lib().pdd_regime_analyse(float(f_min), float(f_max), float(sigma_norm), float(dx),
                                    C.byref(r))
    _check(st, None)
    d = r.as_dict()
    d["hyperbolic"] = bool(d["hyperbolic"])
    return d


def measure_alu_peaks(reps: int = 5) -> dict:
    """FP32 FFMA and shared-memory (LDS.128) throughput of the current device, measured by the
    library's micro-benchmarks (pdd_measure_alu_peaks): the roofline denominators of bench.py."""
    f, m, d = C.c_double(0.0), C.c_double(0.0), C.c_double(0.0)
    _check(N.lib().pdd_measure_alu_peaks(None, int(reps), C.byref(f), C.byref(m), C.byref(d)), None)
    return {"fp32_tflops": f.value, "smem_tbs": m.value, "fp64_tflops": d.value}
