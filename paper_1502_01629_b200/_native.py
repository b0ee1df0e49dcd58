"""ctypes declarations of the C ABI in include/pdd.h (argument marshalling only).

Loads the in-tree ``libpdd.so``; there is no fallback: if the library is missing the import
fails loudly (build it with ``python -m paper_1502_01629_b200.build`` or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpdd.so")


def use_library(path: str) -> None:
    """Development A/B only (scripts/): load another build of the same sources instead of the
    in-tree libpdd.so.  Must be called before the first lib() call."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("libpdd is already loaded")
    LIB_PATH = path

PDD_OK, PDD_E_INVALID, PDD_E_NOCONVERGE, PDD_E_IO, PDD_E_CUDA, PDD_E_STATE, PDD_E_NOMEM, \
    PDD_E_STENCIL = range(8)
STATUS_NAMES = {0: "PDD_OK", 1: "PDD_E_INVALID", 2: "PDD_E_NOCONVERGE", 3: "PDD_E_IO",
                4: "PDD_E_CUDA", 5: "PDD_E_STATE", 6: "PDD_E_NOMEM", 7: "PDD_E_STENCIL"}

EXPORTS = ["pdd_version", "pdd_workspace_bytes", "pdd_create", "pdd_coarse_solve",
           "pdd_synthesize", "pdd_build_patches", "pdd_build_static", "pdd_solve",
           "pdd_apply_operator", "pdd_get_values", "pdd_set_values", "pdd_get_uhat",
           "pdd_get_coarse_values", "pdd_get_controls", "pdd_get_labels", "pdd_get_successors",
           "pdd_get_patch_rounds", "pdd_get_patch_residuals", "pdd_get_tile_rounds",
           "pdd_set_tile_cols", "pdd_set_tile_shape", "pdd_choose_tile_shape", "pdd_kernel_launches", "pdd_last_error", "pdd_destroy",
           "pdd_regime_analyse", "pdd_fuzzy_scratch_bytes", "pdd_build_fuzzy_patches",
           "pdd_fuzzy_sparse_scratch_bytes", "pdd_build_fuzzy_patches_sparse", "pdd_measure_alu_peaks"]


class pdd_coef(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value", C.c_double), ("data", C.POINTER(C.c_double))]


class pdd_problem(C.Structure):
    _fields_ = [("n", C.c_int32), ("lo", C.c_double), ("hi", C.c_double), ("dx", C.c_double),
                ("h", C.c_double), ("lam", C.c_double), ("n_controls", C.c_int32),
                ("controls", C.POINTER(C.c_double)), ("speed", pdd_coef),
                ("drift", pdd_coef * 2), ("p", C.c_int32), ("sigma", (pdd_coef * 2) * 2),
                ("cost", pdd_coef), ("diffusion_scale", C.c_int32),
                ("kind", C.POINTER(C.c_uint8)), ("sector", C.POINTER(C.c_int16)),
                ("sigma_mode", C.c_int32), ("cost_ctrl", C.POINTER(C.c_double))]


class pdd_solve_opts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("k_inner", C.c_int32), ("tol", C.c_double),
                ("max_rounds", C.c_int64), ("delta", C.c_double), ("kernel", C.c_int32),
                ("schedule", C.c_int32), ("early_exit_off", C.c_int32),
                ("bucket_policy", C.c_int32), ("trace", C.c_int32), ("queue_target", C.c_int32)]


class pdd_solve_stats(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("node_updates", C.c_int64),
                ("tiles_processed", C.c_int64), ("verify_passes", C.c_int64),
                ("final_residual", C.c_double), ("apost_bound", C.c_double),
                ("seconds_total", C.c_double), ("seconds_sweep", C.c_double),
                ("seconds_verify", C.c_double), ("converged", C.c_int32),
                ("n_tiles", C.c_int32), ("kernel_used", C.c_int32),
                ("patches_active", C.c_int32), ("patches_converged", C.c_int32),
                ("tile_cols", C.c_int32), ("tile_rows", C.c_int32), ("tiles_x", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class pdd_regime(C.Structure):
    _fields_ = [("omega", C.c_double), ("upsilon", C.c_double), ("alpha_lo", C.c_double),
                ("alpha_hi", C.c_double), ("alpha", C.c_double), ("h", C.c_double),
                ("tau_dx", C.c_double), ("eps_threshold", C.c_double), ("hyperbolic", C.c_int32),
                ("reserved", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class pdd_fuzzy_stats(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("residual", C.c_double), ("seconds", C.c_double),
                ("converged", C.c_int32), ("overlap_nodes", C.c_int32), ("phi_offset", C.c_int64),
                ("lab_offset", C.c_int64), ("max_list", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class pdd_coarse_stats(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("residual", C.c_double), ("seconds", C.c_double),
                ("converged", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libpdd.so not found at {LIB_PATH}: build it first "
                          "(python -m paper_1502_01629_b200.build); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, ctx = C.c_void_p, C.c_void_p
    P = C.POINTER(pdd_problem)
    L.pdd_version.restype = C.c_char_p
    L.pdd_last_error.argtypes = [ctx]
    L.pdd_last_error.restype = C.c_char_p
    L.pdd_workspace_bytes.argtypes = [P, P, C.c_int32, C.POINTER(C.c_size_t)]
    L.pdd_create.argtypes = [P, P, C.c_int32, vp, vp, C.c_size_t, C.POINTER(ctx)]
    L.pdd_coarse_solve.argtypes = [ctx, C.c_double, C.c_int64, C.POINTER(pdd_coarse_stats)]
    L.pdd_synthesize.argtypes = [ctx]
    L.pdd_build_patches.argtypes = [ctx, C.c_int32, C.c_double]
    L.pdd_build_static.argtypes = [ctx, C.c_int32, C.c_int32]
    L.pdd_solve.argtypes = [ctx, C.POINTER(pdd_solve_opts), C.POINTER(pdd_solve_stats)]
    L.pdd_apply_operator.argtypes = [ctx, vp, C.c_int32, C.POINTER(C.c_double)]
    L.pdd_get_values.argtypes = [ctx, vp, C.c_int32, C.c_int32]
    L.pdd_set_values.argtypes = [ctx, vp, C.c_int32]
    for f in ("pdd_get_uhat", "pdd_get_coarse_values", "pdd_get_controls", "pdd_get_labels",
              "pdd_get_successors"):
        getattr(L, f).argtypes = [ctx, vp, C.c_int32]
    L.pdd_get_patch_rounds.argtypes = [ctx, vp, C.c_int32]
    L.pdd_get_patch_residuals.argtypes = [ctx, vp, C.c_int32]
    L.pdd_get_tile_rounds.argtypes = [ctx, vp, C.c_int32]
    L.pdd_set_tile_cols.argtypes = [ctx, C.c_int32]
    L.pdd_set_tile_shape.argtypes = [ctx, C.c_int32, C.c_int32]
    L.pdd_choose_tile_shape.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_int32,
                                        C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.pdd_fuzzy_scratch_bytes.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]
    L.pdd_build_fuzzy_patches.argtypes = [ctx, C.c_int32, C.c_double, C.c_double, C.c_int64, vp,
                                          C.c_size_t, C.POINTER(pdd_fuzzy_stats)]
    L.pdd_measure_alu_peaks.argtypes = [vp, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
    L.pdd_fuzzy_sparse_scratch_bytes.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]
    L.pdd_build_fuzzy_patches_sparse.argtypes = [ctx, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                                 C.c_int64, vp, C.c_size_t, C.POINTER(pdd_fuzzy_stats)]
    L.pdd_regime_analyse.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double,
                                     C.POINTER(pdd_regime)]
    L.pdd_destroy.argtypes = [ctx]
    L.pdd_kernel_launches.argtypes = [ctx]
    L.pdd_kernel_launches.restype = C.c_longlong
    L.pdd_destroy.restype = None
    for f in EXPORTS:
        if f not in ("pdd_version", "pdd_last_error", "pdd_destroy", "pdd_kernel_launches"):
            getattr(L, f).restype = C.c_int
    _lib = L
    return L
