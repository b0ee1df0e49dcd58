"""The lean general-stencil kernel (path 4, csrc/sweep_gf.cuh: coefficient planes in shared
memory, compile-time branch count, self weight removed once per control) against the oracle:
the operator T node by node, and full solves through the work queue, on instances with a speed
field (C3), a row-uniform drift (C5, forced off its row table), x-varying drift fields, one noise
column (C4: two branches), a per-control cost and ragged / boundary tiles (clamped feet)."""
import numpy as np
import pytest

import oracle as O
import pdd_inputs as I

pytestmark = pytest.mark.gpu


def _solver(inst, precision):
    from paper_1502_01629_b200 import Solver
    return Solver(inst, precision=precision)


def _smooth_field(inst, seed):
    rng = np.random.default_rng(seed)
    n = inst.n
    x = inst.x(np.arange(n))
    X, Y = np.meshgrid(x, x, indexing="xy")
    V = (0.4 * np.hypot(X, Y) + 0.05 * np.sin(7 * X) * np.cos(5 * Y)).reshape(-1)
    V = V + 1e-3 * rng.standard_normal(V.size)
    V[inst.kind == I.KIND_TARGET] = 0.0
    V[inst.kind == I.KIND_OBSTACLE] = 1.0 / inst.lam
    return V


def _drift_field_instance(n, p=2, cost_ctrl=False):
    """Speed AND drift vary along x1 (the DRIFTX planes): a swirl about the centre."""
    lo, hi = -1.0, 1.0
    dx = I.grid_params(n, lo, hi)
    x = lo + dx * np.arange(n)
    X, Y = np.meshgrid(x, x, indexing="xy")
    speed = I.Coef.field((1.0 + 0.4 * np.sin(3 * X) * np.cos(2 * Y)).reshape(-1))
    d1 = I.Coef.field((-0.3 * Y / (0.2 + X * X + Y * Y)).reshape(-1))
    d2 = I.Coef.field((0.3 * X / (0.2 + X * X + Y * Y)).reshape(-1))
    s = 0.25 * np.sqrt(dx)
    z = I.Coef.const(0.0)
    sig = ((I.Coef.const(s), z), (z, I.Coef.const(s))) if p == 2 else ((I.Coef.const(s), I.Coef.const(0.5 * s)), (z, z))
    mask, _ = I.ball_target(n, lo, dx, (0.1, -0.2), 0.08)
    kind = np.where(mask, I.KIND_TARGET, I.KIND_FREE).astype(np.uint8)
    kw = {}
    if cost_ctrl:
        a = I.unit_circle_controls(24)
        kw["cost_ctrl"] = 0.3 * np.abs(a[:, 0] / (2.0 + a[:, 1]))
    return I.make_instance(f"swirl{n}", n, lo, hi, n_a=24, lam=1.0, speed=speed, drift=(d1, d2), p=p,
                           sigma=sig, kind=kind, **kw)


CASES = [("C3", 257), ("C3", 300), ("C5", 257), ("C4", 257), ("C2", 201), ("C1", None)]


@pytest.mark.parametrize("cfg,n", CASES)
@pytest.mark.parametrize("precision", [64, 32])
def test_lean_operator_parity(cfg, n, precision):
    inst = I.make_config(cfg, n=n)
    V = _smooth_field(inst, 5)
    ref, _ = O.apply(inst, V)
    s = _solver(inst, precision)
    out, res = s.apply_operator(V, kernel=4)
    err = np.abs(out - ref).max()
    assert err < (1e-12 if precision == 64 else 2e-6 * np.abs(V).max()), err
    assert abs(res - np.abs(ref - V)[inst.kind == 0].max()) < (1e-12 if precision == 64 else 4e-6)
    # and it is the kernel the automatic choice takes for a general-stencil problem
    if cfg == "C3":
        out0, _ = s.apply_operator(V, kernel=0)
        assert np.array_equal(out0, out)
    s.close()


@pytest.mark.parametrize("p,cost_ctrl", [(2, False), (1, False), (2, True)])
@pytest.mark.parametrize("precision", [64, 32])
def test_lean_operator_drift_planes(p, cost_ctrl, precision):
    inst = _drift_field_instance(161, p=p, cost_ctrl=cost_ctrl)
    V = _smooth_field(inst, 9)
    ref, _ = O.apply(inst, V)
    s = _solver(inst, precision)
    out, _ = s.apply_operator(V, kernel=4)
    err = np.abs(out - ref).max()
    assert err < (1e-12 if precision == 64 else 2e-6 * np.abs(V).max()), err
    gen, _ = s.apply_operator(V, kernel=1)           # the fully general kernel agrees too
    assert np.abs(gen - ref).max() < (1e-12 if precision == 64 else 2e-6 * np.abs(V).max())
    s.close()


@pytest.mark.parametrize("precision", [64, 32])
def test_lean_solve_parity_drift_planes(precision):
    inst = _drift_field_instance(161)
    tol_o = 2e-11 * (1.0 - inst.beta)
    ref = O.jacobi(inst, tol=tol_o, max_sweeps=10**6)["V"]
    s = _solver(inst, precision)
    s.build_static(2, 2)
    st = s.solve("static", tol=tol_o if precision == 64 else 1e-7, kernel=4)
    assert st["converged"] == 1 and st["kernel_used"] == 4
    err = np.abs(s.get_values() - ref).max()
    assert err <= (1e-10 if precision == 64 else 5e-5 * np.abs(ref).max()), err
    s.close()


@pytest.mark.parametrize("mode", ["patchy", "static"])
def test_lean_solve_parity_c3(mode):
    """C3 (speed field) at 257^2 through the work queue: the automatic kernel is path 4."""
    inst = I.make_config("C3", n=257)
    ref = O.jacobi(inst, tol=2e-11 * (1.0 - inst.beta), max_sweeps=10**6)["V"]
    s = _solver(inst, 32)
    if mode == "patchy":
        s.coarse_solve(inst.tol_coarse)
        s.synthesize()
        s.build_patches(inst.n_patches)
    else:
        s.build_static(*inst.static_blocks)
    st = s.solve(mode, tol=1e-7)
    assert st["converged"] == 1 and st["kernel_used"] == 4
    assert np.abs(s.get_values() - ref).max() <= 5e-5 * np.abs(ref).max()
    # the rounds schedule runs the fully general kernel (path 1) to the same fixed point
    st1 = s.solve(mode, tol=1e-7, schedule="rounds")
    assert st1["converged"] == 1 and st1["kernel_used"] == 1
    assert np.abs(s.get_values() - ref).max() <= 5e-5 * np.abs(ref).max()
    s.close()


def test_lean_kernel_refused_where_it_does_not_apply():
    from paper_1502_01629_b200 import PddError
    from paper_1502_01629_b200 import _native as N
    inst = I.exit_instance(41, problem="eikonal", eps=1e-3)      # lambda = 0: exit problem
    s = _solver(inst, 64)
    s.build_static(1, 1)
    with pytest.raises(PddError) as e:
        s.solve("static", tol=1e-9, kernel=4)
    assert e.value.status == N.PDD_E_INVALID
    st = s.solve("static", tol=1e-9)                             # automatic: path 1 or 2
    assert st["converged"] == 1 and st["kernel_used"] != 4
    s.close()
